// Internal runtime structures of libgs.so (context, models, requests, per-rank arenas).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <atomic>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/gs.h"
#include "kernels.h"

namespace gs {

using bf16 = __nv_bfloat16;

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

struct BlockW {
  bf16 *w_qkv, *b_qkv, *g_q, *g_k, *w_o, *b_o, *w_1, *b_1, *w_2, *b_2;
  float* mod;  // [6, D]
  // text cross-attention (NEXT-1; null without cross_attn)
  bf16 *ln3_w = nullptr, *ln3_b = nullptr, *w_cq = nullptr, *b_cq = nullptr, *w_ckv = nullptr,
       *b_ckv = nullptr, *g_cq = nullptr, *g_ck = nullptr, *w_co = nullptr, *b_co = nullptr;
  float *ln3_scale_m1 = nullptr, *ln3_shift = nullptr;  // fp32 (ln3_w - 1), ln3_b for ln_modulate
};

struct Model {
  gs_model_desc desc{};
  int hd = 0;  // head dim
  std::vector<BlockW> blocks;
  bf16 *w_pe, *b_pe, *w_t1, *b_t1, *w_t2, *b_t2, *w_tp, *b_tp, *w_head, *b_head;
  bf16 *w_te1 = nullptr, *b_te1 = nullptr, *w_te2 = nullptr, *b_te2 = nullptr;  // text embedding
  float* zeros = nullptr;  // [D] fp32
  float* mod_head;     // [2, D]
  float2* cs_tab;      // [p_max, hd/2]
  int* slot_axis;      // [hd/2]
  int p_max = 1024;
  std::vector<void*> allocs;
};

struct Shard {
  int rank = -1;
  int lo = 0, hi = 0;  // token range
  float* z = nullptr;  // device [hi-lo, lat] fp32 if this process owns `rank`
  size_t bytes = 0;    // pool block size of z
};

struct Request {
  gs_req id = 0;
  int model = 0;
  int grid[3] = {1, 1, 1};
  int n = 0;
  int steps = 0;
  int step_idx = 0;
  int state = GS_REQ_PLACED;
  std::vector<int> ranks;
  std::vector<Shard> shards;  // one per SP position
  std::atomic<int> preempt{0};
  // text conditioning (cross-attention models): nb = 1 (cond) or 2 (cond + uncond, CFG scale cfg)
  int nb = 1;
  float cfg = 0.f;
  uint64_t prompt_seed = 0;
  std::vector<uint16_t> prompt_host;  // [nb][text_len][text_dim] bf16 bits if given by the caller
  // per local rank index: context K / V of every layer [nb][layers][2][text_len][D] bf16
  std::map<int, DevBuf> ctx_kv;
};

// Per-local-rank arena (grow-only device buffers).
struct RankArena {
  int rank = 0;
  DevBuf x, a, qkv, qs, ks, vs, qr, kr, vr, o, orecv, ostage, h, zpack, zb, e0, e, temb, row_req,
      row_tok, req_grid, qc, vbuf;
};

struct Prof {
  double ms = 0;
  long long n = 0;
};

}  // namespace gs

struct gs_ctx {
  int device = 0;
  int world = 1;
  int my_rank = 0;   // real mode
  bool emulated = false;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  ncclComm_t comm = nullptr;
  std::vector<gs::RankArena> local;  // emulated: world entries; real: 1 entry
  std::vector<std::unique_ptr<gs::Model>> models;
  std::map<gs_req, std::unique_ptr<gs::Request>> reqs;
  gs_req next_req = 1;
  std::string err;
  std::mutex table_mu;  // guards reqs
  std::mutex run_mu;    // one run / resume at a time
  // measurement
  bool prof = false;        // per-kernel-class events (gs_profile enable = 1)
  bool prof_steps = false;  // per-step events (enable = 1 or 2)
  std::map<std::string, gs::Prof> prof_tab;
  std::vector<std::pair<std::string, std::pair<cudaEvent_t, cudaEvent_t>>> prof_pending;
  std::vector<cudaEvent_t> event_pool;
  std::vector<float> step_ms;       // device time of each profiled step (gs_stats "step_ms")
  long long launches = 0;
  cudaEvent_t ev_order = nullptr;   // debug entry points: order after the legacy stream
  // caching allocator for per-request state (latent shards, text caches): released blocks are
  // kept for reuse -- submit / release in a serving loop never reach cudaMalloc / cudaFree, whose
  // cost after an idle period was measured at 250-650 ms.  All users are ordered on `stream`.
  std::multimap<size_t, void*> pool;
  // pinned scratch for preemption agreement
  int* h_flag = nullptr;
  int* d_flag = nullptr;
  // fused (peer-store) all-to-alls: mode 1 = peer stores wherever p divides the
  // heads (default), 0 = transfer plans (NCCL send / recv, emulated device copies)
  int a2a_mode = 1;
  unsigned long long* flags = nullptr;                    // [world (emulated) or 1][8] barrier words
  unsigned long long sig_sent[8][8] = {}, sig_seen[8][8] = {};  // per (src, dst) global rank pair
  unsigned long long probe_sent[8] = {}, probe_seen[8] = {};      // NCCL mode: mapping probes per peer
  struct PeerMap {                                        // NCCL mode: CUDA IPC mappings of a peer
    cudaIpcMemHandle_t h[5];                              // qr, kr, vr, orecv, flags
    void* p[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  };
  PeerMap peers[8];
  void* ipc_dev = nullptr;                                // device staging of the handle exchange
  long long a2a_peer = 0, a2a_plan = 0;                   // exchanges run each way (gs_stats)
};
