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
#include <thread>
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

// VAE decoder (NEXT-4, csrc/vae.cpp): modules in the walk order of synth/vae.py (independently
// re-built there); convolution weights padded to [Coutp][kt kh kw][Cp] bf16.
struct VaeConv {
  int cin = 0, cout = 0, kt = 1, kh = 1, kw = 1, cp = 0, coutp = 0;
  __nv_bfloat16* w = nullptr;
  __nv_bfloat16* b = nullptr;
};
struct VaeNorm {
  int c = 0;
  __nv_bfloat16* gamma = nullptr;
};
struct VaeRes {
  VaeNorm n1, n2;
  VaeConv c1, c2, skip;  // skip.cout == 0: identity shortcut
};
struct Vae {
  gs_vae_desc desc{};
  float* mean = nullptr;  // [z_dim] fp32
  float* stdv = nullptr;
  VaeConv post, conv_in, conv_out;
  std::vector<VaeRes> mid;
  std::vector<std::vector<VaeRes>> up;  // per stage
  std::vector<VaeConv> tconv, sconv;    // per stage (tconv.cout == 0: no temporal upsample)
  VaeNorm norm_out;
  std::vector<void*> allocs;
  DevBuf act[4];        // activation buffers (roles X, N, H, S), grow-only across decodes
  DevBuf lat_stage, vid_stage;
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
  // written by a run's worker thread, read by gs_query / gs_preempt on the caller's thread
  std::atomic<int> step_idx{0};
  std::atomic<int> state{GS_REQ_PLACED};
  // a request submitted without placement (GS_REQ_QUEUED) keeps the recipe of its initial latent
  // until gs_place: the noise seed, or the caller's latent copied at submit
  uint64_t noise_seed = 0;
  std::vector<float> init_host;
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
      row_tok, req_grid, qc, vbuf, ssq;
};

struct Prof {
  double ms = 0;
  long long n = 0;
};

// An asynchronous run (gs_run_steps_async): its worker thread, result and GPU set.
struct Ticket {
  std::thread th;
  int rc = GS_OK;
  int steps_run = 0;
  std::string err;
  std::vector<int> ranks;
  std::atomic<int> finished{0};
};

// The stream a thread launches the context's work on: a run's worker thread sets its lane (the
// stream of the run's first rank); API calls use the lane of the ranks they act on, or lane 0.
extern thread_local cudaStream_t tl_stream;
// Error message sink of a worker thread (its ticket); nullptr = the context's message.
extern thread_local std::string* tl_err;

}  // namespace gs

struct gs_ctx {
  int device = 0;
  int world = 1;
  int my_rank = 0;   // real mode
  bool emulated = false;
  int num_sms = 148;
  cudaStream_t stream = nullptr;     // lane 0 (the caller thread's default)
  std::vector<cudaStream_t> lanes;   // per local rank index: stream of runs led by that rank
  ncclComm_t comm = nullptr;
  std::vector<gs::RankArena> local;  // emulated: world entries; real: 1 entry
  std::vector<std::unique_ptr<gs::Model>> models;
  std::vector<std::unique_ptr<gs::Vae>> vaes;
  std::map<gs_req, std::unique_ptr<gs::Request>> reqs;
  gs_req next_req = 1;
  std::string err;
  std::mutex api_mu;    // serialises the API calls that allocate or launch (not the runs' workers)
  std::mutex table_mu;  // guards reqs, request states, tickets, busy
  std::mutex err_mu;    // err
  std::mutex pool_mu;   // pool
  std::mutex prof_mu;   // prof_tab, prof_pending, event_pool, step_ms
  // asynchronous runs: in-flight tickets and, per global rank, the ticket using it (0 = idle);
  // runs on overlapping GPU sets are refused (Eq. capacity; Alg.1 "no GPU overlap")
  std::map<gs_ticket, std::unique_ptr<gs::Ticket>> tickets;
  gs_ticket next_ticket = 1;
  std::vector<gs_ticket> busy;
  // measurement
  bool prof = false;        // per-kernel-class events (gs_profile enable = 1)
  bool prof_steps = false;  // per-step events (enable = 1 or 2)
  std::map<std::string, gs::Prof> prof_tab;
  std::vector<std::pair<std::string, std::pair<cudaEvent_t, cudaEvent_t>>> prof_pending;
  std::vector<cudaEvent_t> event_pool;
  std::vector<float> step_ms;       // device time of each profiled step (gs_stats "step_ms")
  std::atomic<long long> launches{0};
  cudaEvent_t ev_order = nullptr;   // debug entry points: order after the legacy stream
  // caching allocator for per-request state (latent shards, text caches): released blocks are
  // kept for reuse -- submit / release in a serving loop never reach cudaMalloc / cudaFree, whose
  // cost after an idle period was measured at 250-650 ms.  All users are ordered on `stream`.
  std::multimap<size_t, void*> pool;
  // pinned scratch for preemption agreement
  int* h_flag = nullptr;   // [64]: per-step agreement (flag, arena generation) and probe results
  int* d_flag = nullptr;
  // NCCL mode: control-plane communicator (ncclCommSplit of comm) for the job-wide request-id check,
  // so a gs_submit on the caller's thread never drives the communicator a run's worker uses
  ncclComm_t ctrl = nullptr;
  long long* h_id = nullptr;  // [4] scratch of the id check
  long long* d_id = nullptr;
  // fused (peer-store) all-to-alls: mode 1 = peer stores wherever p divides the
  // heads (default), 0 = transfer plans (NCCL send / recv, emulated device copies)
  int a2a_mode = 1;
  // USP hybrid (NEXT-2): ring degree r > 1 runs SP degree p as Ulysses over p / r head
  // groups x a ring of r query chunks per head (K / V gathered in token order; bit-exact with every
  // other degree); applies to batches whose p is a multiple of r with p / r dividing the heads
  int usp_ring = 1;
  unsigned long long* flags = nullptr;                    // [world (emulated) or 1][8] barrier words
  unsigned long long sig_sent[8][8] = {}, sig_seen[8][8] = {};  // per (src, dst) global rank pair
  unsigned long long probe_sent[8] = {}, probe_seen[8] = {};      // NCCL mode: mapping probes per peer
  struct PeerMap {                                        // NCCL mode: CUDA IPC mappings of a peer
    cudaIpcMemHandle_t h[5];                              // qr, kr, vr, orecv, flags
    void* p[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  };
  PeerMap peers[8];
  // IPC mapping cache (NCCL mode): the exported buffers' generation (bumped whenever one of them is
  // re-allocated), and per peer the generation its cached mappings belong to; a run whose SP group
  // reports unchanged generations in the step-0 agreement re-uses the mappings without exchanging
  // handles or probing
  unsigned arena_gen = 1;
  void* exported[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  unsigned peer_gen[8] = {};
  std::vector<int> cached_group;  // ranks of the last verified peer-store group
  bool cached_ok = false;
  long long ipc_exchanges = 0;    // full handle exchanges (gs_stats)
  void* ipc_dev = nullptr;                                // device staging of the handle exchange
  std::atomic<long long> a2a_peer{0}, a2a_plan{0};       // exchanges run each way (gs_stats)
};
