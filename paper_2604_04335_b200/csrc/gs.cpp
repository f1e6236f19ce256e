// libgs.so: C-ABI (include/gs.h) and host runtime of the DiT-step hot path.
//
// Executor for one batched denoising step at SP degree p (SURVEY.md §3 "Ours", §8(a)):
//   time-embed -> patch-embed GEMM -> L x { LN1+mod -> QKV GEMM -> qk-RMSNorm+RoPE+pack ->
//   a2a seq->head -> flash attention -> a2a head->seq -> O GEMM (+gated residual) ->
//   LN2+mod -> MLP-up GEMM (+GELU) -> MLP-down GEMM (+gated residual) } -> head LN+mod ->
//   head GEMM (+Euler update of the latent shard).
// The latent stays token-sharded across steps; preemption is checked at step boundaries;
// resume re-shards by copying contiguous token ranges (interval intersections).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "plan.h"
#include "runtime.h"

using namespace gs;

namespace gs {
thread_local cudaStream_t tl_stream = nullptr;
thread_local std::string* tl_err = nullptr;
}  // namespace gs

namespace {

constexpr int MAX_BATCH = 8;

// The stream this thread launches the context's work on (runtime.h tl_stream).
inline cudaStream_t strm(gs_ctx* c) { return tl_stream ? tl_stream : c->stream; }

int fail(gs_ctx* c, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (tl_err) {
    *tl_err = buf;
  } else if (c) {
    std::lock_guard<std::mutex> g(c->err_mu);
    c->err = buf;
  }
  return code;
}

int no_runs_in_flight(gs_ctx* c, const char* what);

// GS_DEBUG=1: progress lines on stderr (diagnosis of hangs on the GPU box)
bool dbg_on() {
  static const bool on = getenv("GS_DEBUG") != nullptr;
  return on;
}
#define DBG(...)                            \
  do {                                      \
    if (dbg_on()) {                         \
      fprintf(stderr, "[gs] " __VA_ARGS__); \
      fprintf(stderr, "\n");                \
      fflush(stderr);                       \
    }                                       \
  } while (0)

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(c, GS_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_)); \
  } while (0)

#define NK(call)                                                                          \
  do {                                                                                    \
    ncclResult_t r_ = (call);                                                             \
    if (r_ != ncclSuccess)                                                                \
      return fail(c, GS_ENCCL, "%s:%d %s: %s", __FILE__, __LINE__, #call, ncclGetErrorString(r_)); \
  } while (0)

#define RET(call)               \
  do {                          \
    int rc_ = (call);           \
    if (rc_ != GS_OK) return rc_; \
  } while (0)

int ensure(gs_ctx* c, DevBuf& b, size_t bytes) {
  if (bytes <= b.cap) return GS_OK;
  if (b.p) {
    CK(cudaStreamSynchronize(strm(c)));
    CK(cudaFree(b.p));
    b.p = nullptr;
    b.cap = 0;
  }
  size_t want = bytes + bytes / 8 + 256;
  if (cudaMalloc(&b.p, want) != cudaSuccess) {
    cudaGetLastError();
    b.p = nullptr;
    return fail(c, GS_ENOMEM, "cudaMalloc(%zu) failed", want);
  }
  b.cap = want;
  return GS_OK;
}

// ------------------------------------------------------------------ caching allocator
constexpr size_t kPoolGrain = size_t(2) << 20;  // 2 MiB blocks

size_t pool_round(size_t bytes) { return (std::max<size_t>(bytes, 1) + kPoolGrain - 1) / kPoolGrain * kPoolGrain; }

void* pool_alloc(gs_ctx* c, size_t bytes) {
  std::lock_guard<std::mutex> g(c->pool_mu);
  const size_t sz = pool_round(bytes);
  auto it = c->pool.find(sz);
  if (it != c->pool.end()) {
    void* p = it->second;
    c->pool.erase(it);
    return p;
  }
  void* p = nullptr;
  if (cudaMalloc(&p, sz) == cudaSuccess) return p;
  cudaGetLastError();
  cudaStreamSynchronize(strm(c));  // out of memory: return the cached blocks and retry
  for (auto& kv : c->pool) cudaFree(kv.second);
  c->pool.clear();
  if (cudaMalloc(&p, sz) == cudaSuccess) return p;
  cudaGetLastError();
  return nullptr;
}

// Callers free a block only after its last user completed (the owning request is not running and
// the freeing path synchronised its stream), so a block may be reused on any lane.
void pool_free(gs_ctx* c, void* p, size_t bytes) {
  std::lock_guard<std::mutex> g(c->pool_mu);
  if (p) c->pool.emplace(pool_round(bytes), p);
}

// ------------------------------------------------------------------ profiling scopes
cudaEvent_t get_event(gs_ctx* c) {  // caller holds prof_mu
  if (!c->event_pool.empty()) {
    cudaEvent_t e = c->event_pool.back();
    c->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

struct Scope {
  gs_ctx* c;
  const char* name;
  cudaEvent_t a = nullptr, b = nullptr;
  Scope(gs_ctx* c_, const char* n, int launches) : c(c_), name(n) {
    c->launches += launches;
    if (c->prof) {
      std::lock_guard<std::mutex> g(c->prof_mu);
      a = get_event(c);
      b = get_event(c);
      cudaEventRecord(a, strm(c));
    }
  }
  ~Scope() {
    if (c->prof) {
      std::lock_guard<std::mutex> g(c->prof_mu);
      cudaEventRecord(b, strm(c));
      c->prof_pending.push_back({name, {a, b}});
    }
  }
};

void prof_flush(gs_ctx* c) {
  std::lock_guard<std::mutex> g(c->prof_mu);
  // "_gaps": device time between consecutive scopes (launch latency, kernel ramp / drain outside
  // any kernel, host-side stalls), = span(first start .. last end) - sum of the scopes.
  if (c->prof_pending.size() > 1) {
    float span = 0, inside = 0;
    cudaEventElapsedTime(&span, c->prof_pending.front().second.first, c->prof_pending.back().second.second);
    for (auto& pe : c->prof_pending) {
      float ms = 0;
      cudaEventElapsedTime(&ms, pe.second.first, pe.second.second);
      inside += ms;
    }
    auto& g = c->prof_tab["_gaps"];
    g.ms += span - inside;
    g.n += 1;
  }
  for (auto& pe : c->prof_pending) {
    float ms = 0;
    cudaEventElapsedTime(&ms, pe.second.first, pe.second.second);
    auto& p = c->prof_tab[pe.first];
    p.ms += ms;
    p.n += 1;
    c->event_pool.push_back(pe.second.first);
    c->event_pool.push_back(pe.second.second);
  }
  c->prof_pending.clear();
}

int local_index(gs_ctx* c, int rank) {
  if (c->emulated) return (rank >= 0 && rank < c->world) ? rank : -1;
  return rank == c->my_rank ? 0 : -1;
}

double sigma_at(int i, int S, double shift) {
  const double u = 1.0 - static_cast<double>(i) / S;
  return shift * u / (1.0 + (shift - 1.0) * u);
}

bool valid_p(int p) { return p == 1 || p == 2 || p == 4 || p == 8; }

int check_ranks(gs_ctx* c, const int* ranks, int n) {
  if (!ranks || !valid_p(n)) return fail(c, GS_EINVAL, "SP degree %d not in {1,2,4,8}", n);
  for (int i = 0; i < n; ++i) {
    if (ranks[i] < 0 || ranks[i] >= c->world) return fail(c, GS_EINVAL, "rank %d out of range", ranks[i]);
    for (int j = 0; j < i; ++j)
      if (ranks[i] == ranks[j]) return fail(c, GS_EINVAL, "duplicate rank %d", ranks[i]);
  }
  return GS_OK;
}

// ------------------------------------------------------------------ weights
struct WSpec {
  const char* name;
  uint32_t tid;
  int kind;
  long long rows, cols;  // elements = rows * cols
  int fan_in;            // > 0: scale sqrt(3/fan_in)
  float scale;
};

int gen(gs_ctx* c, Model& m, void** dst, const WSpec& s, uint64_t seed) {
  const long long n = s.rows * s.cols;
  const size_t bytes = n * (s.kind == RNG_F32_SCALED ? 4 : 2);
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    return fail(c, GS_ENOMEM, "weight alloc %s (%zu B) failed", s.name, bytes);
  }
  m.allocs.push_back(p);
  const float scale = s.fan_in > 0 ? static_cast<float>(std::sqrt(3.0 / s.fan_in)) : s.scale;
  CK(rng_fill(p, n, seed, s.tid, s.kind, scale, strm(c)));
  *dst = p;
  return GS_OK;
}

// Tensor table of one block / the global parameters (names and tensor ids match synth/rng.py TID).
std::vector<WSpec> block_specs(const gs_model_desc& d) {
  const long long D = d.dim, F = d.ffn;
  return {
      {"w_qkv", 1, RNG_BF16_SCALED, 3 * D, D, (int)D, 0},
      {"b_qkv", 2, RNG_BF16_SCALED, 1, 3 * D, 0, 0.1f},
      {"g_q", 3, RNG_BF16_GAIN, 1, D, 0, 0},
      {"g_k", 4, RNG_BF16_GAIN, 1, D, 0, 0},
      {"w_o", 5, RNG_BF16_SCALED, D, D, (int)D, 0},
      {"b_o", 6, RNG_BF16_SCALED, 1, D, 0, 0.1f},
      {"w_1", 7, RNG_BF16_SCALED, F, D, (int)D, 0},
      {"b_1", 8, RNG_BF16_SCALED, 1, F, 0, 0.1f},
      {"w_2", 9, RNG_BF16_SCALED, D, F, (int)F, 0},
      {"b_2", 10, RNG_BF16_SCALED, 1, D, 0, 0.1f},
      {"mod", 11, RNG_F32_SCALED, 6, D, 0, 0.5f},
  };
}
// Text cross-attention tensors (tensor ids as synth/rng.py TID)
std::vector<WSpec> cross_specs(const gs_model_desc& d) {
  const long long D = d.dim;
  return {
      {"ln3_w", 12, RNG_BF16_GAIN, 1, D, 0, 0},
      {"ln3_b", 13, RNG_BF16_SCALED, 1, D, 0, 0.1f},
      {"w_cq", 14, RNG_BF16_SCALED, D, D, (int)D, 0},
      {"b_cq", 15, RNG_BF16_SCALED, 1, D, 0, 0.1f},
      {"w_ckv", 16, RNG_BF16_SCALED, 2 * D, D, (int)D, 0},
      {"b_ckv", 17, RNG_BF16_SCALED, 1, 2 * D, 0, 0.1f},
      {"g_cq", 18, RNG_BF16_GAIN, 1, D, 0, 0},
      {"g_ck", 19, RNG_BF16_GAIN, 1, D, 0, 0},
      {"w_co", 32, RNG_BF16_SCALED, D, D, (int)D, 0},
      {"b_co", 33, RNG_BF16_SCALED, 1, D, 0, 0.1f},
  };
}
std::vector<WSpec> text_specs(const gs_model_desc& d) {
  const long long D = d.dim, T = d.text_dim;
  return {
      {"w_te1", 40, RNG_BF16_SCALED, D, T, (int)T, 0},
      {"b_te1", 41, RNG_BF16_SCALED, 1, D, 0, 0.1f},
      {"w_te2", 42, RNG_BF16_SCALED, D, D, (int)D, 0},
      {"b_te2", 43, RNG_BF16_SCALED, 1, D, 0, 0.1f},
  };
}
std::vector<WSpec> all_block_specs(const gs_model_desc& d) {
  auto v = block_specs(d);
  if (d.cross_attn)
    for (auto& x : cross_specs(d)) v.push_back(x);
  return v;
}
std::vector<WSpec> global_specs(const gs_model_desc& d) {
  const long long D = d.dim, P = d.lat, T = d.freq_dim;
  return {
      {"w_pe", 20, RNG_BF16_SCALED, D, P, (int)P, 0},
      {"b_pe", 21, RNG_BF16_SCALED, 1, D, 0, 0.1f},
      {"w_t1", 22, RNG_BF16_SCALED, D, T, (int)T, 0},
      {"b_t1", 23, RNG_BF16_SCALED, 1, D, 0, 0.1f},
      {"w_t2", 24, RNG_BF16_SCALED, D, D, (int)D, 0},
      {"b_t2", 25, RNG_BF16_SCALED, 1, D, 0, 0.1f},
      {"w_tp", 26, RNG_BF16_SCALED, 6 * D, D, (int)D, 0},
      {"b_tp", 27, RNG_BF16_SCALED, 1, 6 * D, 0, 0.1f},
      {"mod_head", 28, RNG_F32_SCALED, 2, D, 0, 0.5f},
      {"w_head", 29, RNG_BF16_SCALED, P, D, (int)D, 0},
      {"b_head", 30, RNG_BF16_SCALED, 1, P, 0, 0.1f},
  };
}

std::vector<WSpec> all_global_specs(const gs_model_desc& d) {
  auto v = global_specs(d);
  if (d.cross_attn)
    for (auto& x : text_specs(d)) v.push_back(x);
  return v;
}

void** block_slot(BlockW& b, const char* name) {
  if (!strcmp(name, "w_qkv")) return (void**)&b.w_qkv;
  if (!strcmp(name, "b_qkv")) return (void**)&b.b_qkv;
  if (!strcmp(name, "g_q")) return (void**)&b.g_q;
  if (!strcmp(name, "g_k")) return (void**)&b.g_k;
  if (!strcmp(name, "w_o")) return (void**)&b.w_o;
  if (!strcmp(name, "b_o")) return (void**)&b.b_o;
  if (!strcmp(name, "w_1")) return (void**)&b.w_1;
  if (!strcmp(name, "b_1")) return (void**)&b.b_1;
  if (!strcmp(name, "w_2")) return (void**)&b.w_2;
  if (!strcmp(name, "b_2")) return (void**)&b.b_2;
  if (!strcmp(name, "mod")) return (void**)&b.mod;
  if (!strcmp(name, "ln3_w")) return (void**)&b.ln3_w;
  if (!strcmp(name, "ln3_b")) return (void**)&b.ln3_b;
  if (!strcmp(name, "w_cq")) return (void**)&b.w_cq;
  if (!strcmp(name, "b_cq")) return (void**)&b.b_cq;
  if (!strcmp(name, "w_ckv")) return (void**)&b.w_ckv;
  if (!strcmp(name, "b_ckv")) return (void**)&b.b_ckv;
  if (!strcmp(name, "g_cq")) return (void**)&b.g_cq;
  if (!strcmp(name, "g_ck")) return (void**)&b.g_ck;
  if (!strcmp(name, "w_co")) return (void**)&b.w_co;
  if (!strcmp(name, "b_co")) return (void**)&b.b_co;
  return nullptr;
}
void** global_slot(Model& m, const char* name) {
  if (!strcmp(name, "w_pe")) return (void**)&m.w_pe;
  if (!strcmp(name, "b_pe")) return (void**)&m.b_pe;
  if (!strcmp(name, "w_t1")) return (void**)&m.w_t1;
  if (!strcmp(name, "b_t1")) return (void**)&m.b_t1;
  if (!strcmp(name, "w_t2")) return (void**)&m.w_t2;
  if (!strcmp(name, "b_t2")) return (void**)&m.b_t2;
  if (!strcmp(name, "w_tp")) return (void**)&m.w_tp;
  if (!strcmp(name, "b_tp")) return (void**)&m.b_tp;
  if (!strcmp(name, "mod_head")) return (void**)&m.mod_head;
  if (!strcmp(name, "w_head")) return (void**)&m.w_head;
  if (!strcmp(name, "b_head")) return (void**)&m.b_head;
  if (!strcmp(name, "w_te1")) return (void**)&m.w_te1;
  if (!strcmp(name, "b_te1")) return (void**)&m.b_te1;
  if (!strcmp(name, "w_te2")) return (void**)&m.w_te2;
  if (!strcmp(name, "b_te2")) return (void**)&m.b_te2;
  return nullptr;
}

// ------------------------------------------------------------------ batch plan
// A step's batch.  Rows are laid out per *sequence*: a request, or with classifier-free guidance
// each of its two branches (cond, uncond), which share the latent and timestep but attend only
// within their own branch and to their own prompt.  Row maps point at the request (`real`), so
// time embedding, modulation, gates, RoPE grid and sigma are per request.
struct Plan : A2aGeometry {
  int D = 0, F = 0;
  Model* m = nullptr;
  std::vector<Request*> reqs;    // per sequence
  std::vector<int> branch;       // CFG branch of each sequence (0 = cond, 1 = uncond)
  std::vector<int> real;         // index of the sequence's request in ureqs
  std::vector<Request*> ureqs;   // the batch's requests
  std::vector<int> ranks;
  bool text = false;
  // fused exchange (peer stores): per position its RECV / ORECV buffers and barrier flag words,
  // addressed from this process (local arenas, or CUDA IPC mappings of the peers' buffers)
  bool peer = false;
  std::vector<bf16*> qr_of, kr_of, vr_of, orecv_of;
  std::vector<unsigned long long*> flags_of;
};

void make_plan(Plan& P, Model* m, const std::vector<Request*>& ureqs, const int* ranks, int p, int ring = 1) {
  P.text = m->desc.cross_attn != 0;
  P.ureqs = ureqs;
  P.reqs.clear();
  P.branch.clear();
  P.real.clear();
  for (size_t r = 0; r < ureqs.size(); ++r)
    for (int b = 0; b < (P.text ? ureqs[r]->nb : 1); ++b) {
      P.reqs.push_back(ureqs[r]);
      P.branch.push_back(b);
      P.real.push_back(static_cast<int>(r));
    }
  std::vector<int> n(P.reqs.size());
  for (size_t v = 0; v < P.reqs.size(); ++v) n[v] = P.reqs[v]->n;
  P.init(p, n.data(), static_cast<int>(n.size()), m->desc.heads, m->hd, ring);
  P.m = m;
  P.D = m->desc.dim;
  P.F = m->desc.ffn;
  P.ranks.assign(ranks, ranks + p);
}

// Size the arena of position i and upload its row maps.
int prepare_rank(gs_ctx* c, const Plan& P, int i, RankArena& A) {
  const size_t rows = std::max(P.rows[i], 1), rf = std::max(P.rows_full, 1);
  const size_t D = P.D, F = P.F, lat = P.m->desc.lat;

  RET(ensure(c, A.x, rows * D * 4));
  RET(ensure(c, A.a, rows * D * 2));
  RET(ensure(c, A.qkv, rows * 3 * D * 2));
  if (qk_uses_ssq(D)) RET(ensure(c, A.ssq, rows * (2 * D / 32) * 4));  // QKV GEMM sums of squares of q | k
  RET(ensure(c, A.qs, rows * D * 2));
  RET(ensure(c, A.ks, rows * D * 2));
  RET(ensure(c, A.vs, rows * D * 2));
  (void)rf;
  if (P.p > 1) {
    // receive layouts of A2aGeometry: full heads, then the position's partial-head units
    RET(ensure(c, A.qr, std::max<size_t>(P.recv_q_elems(i), 1) * 2));
    RET(ensure(c, A.kr, std::max<size_t>(P.recv_kv_elems(i), 1) * 2));
    RET(ensure(c, A.vr, std::max<size_t>(P.recv_kv_elems(i), 1) * 2));
    RET(ensure(c, A.o, std::max<size_t>(P.recv_q_elems(i), 1) * 2));
    RET(ensure(c, A.orecv, rows * D * 2));
    RET(ensure(c, A.ostage, rows * D * 2));
  } else {
    RET(ensure(c, A.o, rows * D * 2));
  }
  RET(ensure(c, A.h, rows * F * 2));
  RET(ensure(c, A.zpack, rows * lat * 4));
  if (P.text) {
    RET(ensure(c, A.qc, rows * D * 2));
    RET(ensure(c, A.vbuf, rows * lat * 4));
  }
  RET(ensure(c, A.zb, rows * lat * 2));
  RET(ensure(c, A.e0, MAX_BATCH * D * 4));
  RET(ensure(c, A.e, MAX_BATCH * 6 * D * 4));
  RET(ensure(c, A.temb, (MAX_BATCH * P.m->desc.freq_dim + 2 * MAX_BATCH * D) * 4));
  RET(ensure(c, A.row_req, rows * 4));
  RET(ensure(c, A.row_tok, rows * 4));
  RET(ensure(c, A.req_grid, MAX_BATCH * 3 * 4));
  std::vector<int> rr(P.rows[i]), rt(P.rows[i]), grid(P.ureqs.size() * 3);
  for (int r = 0; r < P.B; ++r)
    for (int t = P.lo[i][r]; t < P.hi[i][r]; ++t) {
      rr[P.loff[i][r] + t - P.lo[i][r]] = P.real[r];
      rt[P.loff[i][r] + t - P.lo[i][r]] = t;
    }
  for (size_t r = 0; r < P.ureqs.size(); ++r)
    for (int a = 0; a < 3; ++a) grid[3 * r + a] = P.ureqs[r]->grid[a];
  if (P.rows[i] > 0) {
    CK(cudaMemcpyAsync(A.row_req.p, rr.data(), rr.size() * 4, cudaMemcpyHostToDevice, strm(c)));
    CK(cudaMemcpyAsync(A.row_tok.p, rt.data(), rt.size() * 4, cudaMemcpyHostToDevice, strm(c)));
  }
  CK(cudaMemcpyAsync(A.req_grid.p, grid.data(), grid.size() * 4, cudaMemcpyHostToDevice, strm(c)));
  CK(cudaStreamSynchronize(strm(c)));  // host vectors go out of scope
  return GS_OK;
}

// gather (dir = 0) / scatter (dir = 1) request shards <-> packed latent of position i
int move_latent(gs_ctx* c, const Plan& P, int i, RankArena& A, int dir) {
  const size_t lat = P.m->desc.lat;
  for (int r = 0; r < P.B; ++r) {
    const size_t cnt = static_cast<size_t>(P.hi[i][r] - P.lo[i][r]) * lat * 4;
    if (!cnt || (dir == 1 && P.branch[r] != 0)) continue;  // the cond rows carry the CFG update
    float* packed = A.zpack.as<float>() + static_cast<size_t>(P.loff[i][r]) * lat;
    float* shard = P.reqs[r]->shards[i].z;
    if (dir == 0)
      CK(cudaMemcpyAsync(packed, shard, cnt, cudaMemcpyDeviceToDevice, strm(c)));
    else
      CK(cudaMemcpyAsync(shard, packed, cnt, cudaMemcpyDeviceToDevice, strm(c)));
  }
  return GS_OK;
}

// ------------------------------------------------------------------ exchanges
// Executors of the host plans (plan.cpp).  NCCL mode: this process is one SP position; sends and
// recvs of the plan go into one NCCL group on the context stream (NVLink / NVSwitch), local
// copies are device copies.  Emulated mode: every position is local; the n-th send of i to j is
// the n-th recv of j from i (the NCCL matching rule), executed as a device copy.
int my_position(gs_ctx* c, const Plan& P) {
  for (int i = 0; i < P.p; ++i)
    if (P.ranks[i] == c->my_rank) return i;
  return -1;
}

int copy_block(gs_ctx* c, void* dst, const void* src, const gs_xfer& x, size_t esz) {
  if (x.rows == 1 || (x.src_pitch == x.width && x.dst_pitch == x.width))
    CK(cudaMemcpyAsync(dst, src, static_cast<size_t>(x.rows * x.width) * esz, cudaMemcpyDeviceToDevice, strm(c)));
  else
    CK(cudaMemcpy2DAsync(dst, x.dst_pitch * esz, src, x.src_pitch * esz, x.width * esz, x.rows,
                         cudaMemcpyDeviceToDevice, strm(c)));
  return GS_OK;
}

// bufs(pos, id) -> base pointer of buffer id of position pos (nullptr if not applicable)
template <class BufFn>
int run_emulated(gs_ctx* c, const std::vector<std::vector<gs_xfer>>& plans, BufFn bufs, size_t esz) {
  const int p = static_cast<int>(plans.size());
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j) {
      if (i == j) continue;
      std::vector<const gs_xfer*> snd, rcv;
      for (const gs_xfer& x : plans[i])
        if (x.op == GS_XFER_SEND && x.peer == j) snd.push_back(&x);
      for (const gs_xfer& x : plans[j])
        if (x.op == GS_XFER_RECV && x.peer == i) rcv.push_back(&x);
      if (snd.size() != rcv.size()) return fail(c, GS_ESTATE, "exchange plan mismatch %d -> %d", i, j);
      for (size_t k = 0; k < snd.size(); ++k) {
        if (snd[k]->width != rcv[k]->width) return fail(c, GS_ESTATE, "exchange size mismatch %d -> %d", i, j);
        char* dst = static_cast<char*>(bufs(j, rcv[k]->dst_buf)) + rcv[k]->dst_off * esz;
        const char* src = static_cast<const char*>(bufs(i, snd[k]->src_buf)) + snd[k]->src_off * esz;
        CK(cudaMemcpyAsync(dst, src, snd[k]->width * esz, cudaMemcpyDeviceToDevice, strm(c)));
      }
    }
  for (int i = 0; i < p; ++i)
    for (const gs_xfer& x : plans[i])
      if (x.op == GS_XFER_COPY)
        RET(copy_block(c, static_cast<char*>(bufs(i, x.dst_buf)) + x.dst_off * esz,
                       static_cast<const char*>(bufs(i, x.src_buf)) + x.src_off * esz, x, esz));
  return GS_OK;
}

// seq -> head: Q/K/V chunk j of position i (rows of i, heads of j) -> recv buffers of j.
int exchange_qkv(gs_ctx* c, const Plan& P) {
  Scope sc(c, "a2a_qkv", 0);
  ++c->a2a_plan;
  // t = 0: Q (plan_q), t = 1, 2: K, V (plan_kv); they differ only for partial-head units
  if (c->emulated) {
    std::vector<std::vector<gs_xfer>> qplans(P.p), kvplans(P.p);
    for (int i = 0; i < P.p; ++i) {
      plan_q(P, i, qplans[i]);
      plan_kv(P, i, kvplans[i]);
    }
    for (int t = 0; t < 3; ++t) {
      auto bufs = [&](int pos, int id) -> void* {
        RankArena& A = c->local[P.ranks[pos]];
        if (id == GS_BUF_SEND) return t == 0 ? A.qs.p : t == 1 ? A.ks.p : A.vs.p;
        return t == 0 ? A.qr.p : t == 1 ? A.kr.p : A.vr.p;
      };
      RET(run_emulated(c, t == 0 ? qplans : kvplans, bufs, 2));
    }
    return GS_OK;
  }
  const int me = my_position(c, P);
  std::vector<gs_xfer> plans[2];
  plan_q(P, me, plans[0]);
  plan_kv(P, me, plans[1]);
  RankArena& A = c->local[0];
  bf16* snd[3] = {A.qs.as<bf16>(), A.ks.as<bf16>(), A.vs.as<bf16>()};
  bf16* rcv[3] = {A.qr.as<bf16>(), A.kr.as<bf16>(), A.vr.as<bf16>()};
  NK(ncclGroupStart());
  for (int t = 0; t < 3; ++t)
    for (const gs_xfer& x : plans[t ? 1 : 0]) {
      if (x.op == GS_XFER_SEND)
        NK(ncclSend(snd[t] + x.src_off, x.width * 2, ncclUint8, P.ranks[x.peer], c->comm, strm(c)));
      else if (x.op == GS_XFER_RECV)
        NK(ncclRecv(rcv[t] + x.dst_off, x.width * 2, ncclUint8, P.ranks[x.peer], c->comm, strm(c)));
    }
  NK(ncclGroupEnd());
  for (int t = 0; t < 3; ++t)
    for (const gs_xfer& x : plans[t ? 1 : 0])
      if (x.op == GS_XFER_COPY) RET(copy_block(c, rcv[t] + x.dst_off, snd[t] + x.src_off, x, 2));
  return GS_OK;
}

// head -> seq: attention output of position j (all rows, heads of j) -> rows' owners.
int exchange_o(gs_ctx* c, const Plan& P) {
  Scope sc(c, "a2a_o", 0);
  ++c->a2a_plan;
  auto arena_buf = [&](RankArena& A, int id) -> void* {
    return id == GS_BUF_O ? A.o.p : id == GS_BUF_STAGE ? A.ostage.p : A.orecv.p;
  };
  if (c->emulated) {
    std::vector<std::vector<gs_xfer>> plans(P.p);
    for (int i = 0; i < P.p; ++i) plan_o(P, i, plans[i], nullptr);
    auto bufs = [&](int pos, int id) -> void* { return arena_buf(c->local[P.ranks[pos]], id); };
    return run_emulated(c, plans, bufs, 2);
  }
  const int me = my_position(c, P);
  std::vector<gs_xfer> plan;
  plan_o(P, me, plan, nullptr);
  RankArena& A = c->local[0];
  NK(ncclGroupStart());
  for (const gs_xfer& x : plan) {
    if (x.op == GS_XFER_SEND)
      NK(ncclSend(static_cast<bf16*>(arena_buf(A, x.src_buf)) + x.src_off, x.width * 2, ncclUint8, P.ranks[x.peer],
                  c->comm, strm(c)));
    else if (x.op == GS_XFER_RECV)
      NK(ncclRecv(static_cast<bf16*>(arena_buf(A, x.dst_buf)) + x.dst_off, x.width * 2, ncclUint8, P.ranks[x.peer],
                  c->comm, strm(c)));
  }
  NK(ncclGroupEnd());
  for (const gs_xfer& x : plan)
    if (x.op == GS_XFER_COPY)
      RET(copy_block(c, static_cast<bf16*>(arena_buf(A, x.dst_buf)) + x.dst_off,
                     static_cast<bf16*>(arena_buf(A, x.src_buf)) + x.src_off, x, 2));
  return GS_OK;
}

// ------------------------------------------------------------------ fused exchange (peer stores)
// The QKV pack kernel stores each head chunk straight into the RECV buffer of the position that
// attends over it, and the attention kernel stores each output row straight into the O-proj input
// (ORECV) of the token's owner: no send / stage buffers, no unpack copies, no NCCL kernels, and the
// NVLink traffic overlaps the producing kernels.  Between producer and consumer a flag barrier
// (peer_signal / peer_wait kernels, system-scope release / acquire) orders the stores; two per
// block (after the pack, after attention) also make every buffer reuse safe: a position writes a
// peer's RECV (ORECV) of layer l + 1 only after that peer passed the barrier that follows its own
// reads of layer l.  Requires p | H (full heads only); other batches use the transfer plans.
struct IpcExport {
  cudaIpcMemHandle_t h[5];
  int ok;
};

int peer_setup(gs_ctx* c, Plan& P, const unsigned* gens = nullptr) {
  P.peer = false;
  if (c->a2a_mode != 1 || P.p == 1 || P.R != 0 || P.B > OSC_MAX_REQ || c->world > 8) return GS_OK;
  P.qr_of.assign(P.p, nullptr);
  P.kr_of.assign(P.p, nullptr);
  P.vr_of.assign(P.p, nullptr);
  P.orecv_of.assign(P.p, nullptr);
  P.flags_of.assign(P.p, nullptr);
  if (c->emulated) {
    for (int j = 0; j < P.p; ++j) {
      RankArena& A = c->local[P.ranks[j]];
      P.qr_of[j] = A.qr.as<bf16>();
      P.kr_of[j] = A.kr.as<bf16>();
      P.vr_of[j] = A.vr.as<bf16>();
      P.orecv_of[j] = A.orecv.as<bf16>();
      P.flags_of[j] = c->flags + static_cast<size_t>(P.ranks[j]) * 16;
    }
    P.peer = true;
    return GS_OK;
  }
  // NCCL mode: exchange CUDA IPC handles of the four buffers and the flag words with the plan's
  // peers (re-opened only when a peer re-allocated), then agree that every position mapped all
  // of them before any kernel stores into peer memory.
  const int me = my_position(c, P);
  if (me < 0) return fail(c, GS_ESTATE, "peer_setup: this process is not in the SP group");
  RankArena& A = c->local[0];
  IpcExport mine{};
  void* bases[5] = {A.qr.p, A.kr.p, A.vr.p, A.orecv.p, c->flags};
  // the arena generation moves whenever an exported buffer was re-allocated since the last run
  if (memcmp(bases, c->exported, sizeof bases) != 0) {
    memcpy(c->exported, bases, sizeof bases);
    ++c->arena_gen;
  }
  auto use_mappings = [&] {
    for (int j = 0; j < P.p; ++j) {
      void* const* p = j == me ? bases : c->peers[P.ranks[j]].p;
      P.qr_of[j] = static_cast<bf16*>(p[0]);
      P.kr_of[j] = static_cast<bf16*>(p[1]);
      P.vr_of[j] = static_cast<bf16*>(p[2]);
      P.orecv_of[j] = static_cast<bf16*>(p[3]);
      P.flags_of[j] = static_cast<unsigned long long*>(p[4]);
    }
    P.peer = true;
  };
  // cache hit: the same SP group verified its mappings before, and every position (this one
  // included, gens from the step-0 agreement) still has the generation those mappings belong to
  if (gens && c->cached_ok && c->cached_group == P.ranks) {
    bool same = gens[me] == c->peer_gen[c->my_rank];
    for (int j = 0; j < P.p && same; ++j)
      if (j != me) same = gens[j] == c->peer_gen[P.ranks[j]];
    if (same) {
      use_mappings();
      return GS_OK;
    }
  }
  ++c->ipc_exchanges;
  for (int b = 0; b < 5; ++b) CK(cudaIpcGetMemHandle(&mine.h[b], bases[b]));
  mine.ok = 1;
  if (!c->ipc_dev) CK(cudaMalloc(&c->ipc_dev, 9 * sizeof(IpcExport)));
  IpcExport* dev = static_cast<IpcExport*>(c->ipc_dev);
  auto exchange = [&](IpcExport* host_all) -> int {
    CK(cudaMemcpyAsync(dev + me, host_all + me, sizeof(IpcExport), cudaMemcpyHostToDevice, strm(c)));
    NK(ncclGroupStart());
    for (int j = 0; j < P.p; ++j) {
      if (j == me) continue;
      NK(ncclSend(dev + me, sizeof(IpcExport), ncclUint8, P.ranks[j], c->comm, strm(c)));
      NK(ncclRecv(dev + j, sizeof(IpcExport), ncclUint8, P.ranks[j], c->comm, strm(c)));
    }
    NK(ncclGroupEnd());
    CK(cudaMemcpyAsync(host_all, dev, P.p * sizeof(IpcExport), cudaMemcpyDeviceToHost, strm(c)));
    CK(cudaStreamSynchronize(strm(c)));
    return GS_OK;
  };
  std::vector<IpcExport> all(P.p);
  all[me] = mine;
  RET(exchange(all.data()));
  int ok = 1;
  for (int j = 0; j < P.p && ok; ++j) {
    if (j == me) continue;
    gs_ctx::PeerMap& pm = c->peers[P.ranks[j]];
    for (int b = 0; b < 5 && ok; ++b) {
      if (pm.p[b] && memcmp(&pm.h[b], &all[j].h[b], sizeof(cudaIpcMemHandle_t)) == 0) continue;
      if (pm.p[b]) cudaIpcCloseMemHandle(pm.p[b]);
      pm.p[b] = nullptr;
      if (cudaIpcOpenMemHandle(&pm.p[b], all[j].h[b], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        pm.p[b] = nullptr;
        ok = 0;
      } else {
        pm.h[b] = all[j].h[b];
      }
    }
  }
  // probe the mappings: store a per-pair counter into every peer's probe word through them and
  // wait (bounded) for every peer's store into ours; then agree -- peer stores only if every
  // position mapped and reached every peer (else the whole group uses the transfer plans)
  if (ok) {
    PeerFlags sig{}, wt{};
    for (int j = 0; j < P.p; ++j) {
      if (j == me) continue;
      const int gj = P.ranks[j];
      sig.slot[sig.n] = static_cast<unsigned long long*>(c->peers[gj].p[4]) + 8 + c->my_rank;
      sig.val[sig.n++] = ++c->probe_sent[gj];
      wt.slot[wt.n] = c->flags + 8 + gj;
      wt.val[wt.n++] = c->probe_seen[gj] + 1;
    }
    CK(peer_signal(sig, strm(c)));
    // probe result in word 40 (words 0-17 carry the per-step agreement)
    CK(peer_wait_probe(wt, 2000, c->d_flag + 40, strm(c)));
    CK(cudaMemcpyAsync(c->h_flag + 40, c->d_flag + 40, 4, cudaMemcpyDeviceToHost, strm(c)));
    CK(cudaStreamSynchronize(strm(c)));
    ok = c->h_flag[40];
    if (ok)
      for (int j = 0; j < P.p; ++j)
        if (j != me) ++c->probe_seen[P.ranks[j]];
  }
  std::vector<IpcExport> agree(P.p);
  agree[me].ok = ok;
  RET(exchange(agree.data()));
  for (int j = 0; j < P.p; ++j) ok &= agree[j].ok;
  c->cached_ok = false;
  if (!ok) return GS_OK;
  use_mappings();
  if (gens) {  // remember the verified group and the generations its mappings belong to
    c->cached_group = P.ranks;
    for (int j = 0; j < P.p; ++j) c->peer_gen[P.ranks[j]] = gens[j];
    c->cached_ok = true;
  }
  return GS_OK;
}

// Flag barrier over the plan's positions (the ones this process owns signal / wait; emulated mode
// signals for every position before any waits, so one stream can carry all of them).  Position
// i tells j "my stores into you are done" by raising word [rank i] of j's flags to the number of
// barriers the pair (i, j) has passed.
int peer_barrier(gs_ctx* c, const Plan& P, const std::vector<int>& mine) {
  Scope sc(c, "a2a_peer_barrier", 2 * static_cast<int>(mine.size()));
  for (int i : mine) {
    PeerFlags f{};
    for (int j = 0; j < P.p; ++j) {
      if (j == i) continue;
      f.slot[f.n] = P.flags_of[j] + P.ranks[i];
      f.val[f.n] = ++c->sig_sent[P.ranks[i]][P.ranks[j]];
      ++f.n;
    }
    CK(peer_signal(f, strm(c)));
  }
  for (int j : mine) {
    PeerFlags f{};
    for (int i = 0; i < P.p; ++i) {
      if (i == j) continue;
      f.slot[f.n] = P.flags_of[j] + P.ranks[i];
      f.val[f.n] = ++c->sig_seen[P.ranks[i]][P.ranks[j]];
      ++f.n;
    }
    CK(peer_wait(f, strm(c)));
  }
  ++c->a2a_peer;
  return GS_OK;
}

// ------------------------------------------------------------------ one step
int gemm(gs_ctx* c, const char* name, int epi, int M, int N, int K, const void* A, const void* W,
         const EpiParams& ep) {
  if (M == 0) return GS_OK;
  Scope sc(c, name, 1);
  CK(gemm_bf16_tc(epi, M, N, K, A, K, W, K, ep, c->num_sms, strm(c)));
  return GS_OK;
}

EpiParams epi(void* out, int ldo, const bf16* bias) {
  EpiParams e{};
  e.out = out;
  e.ldo = ldo;
  e.bias = bias;
  return e;
}

// Pre-attention part of layer l (or the step prologue when l < 0) for position i.
int block_pre(gs_ctx* c, const Plan& P, int i, RankArena& A, int l) {
  const int M = P.rows[i], D = P.D;
  const BlockW& w = P.m->blocks[l];
  const float eps = P.m->desc.eps;
  {
    Scope sc(c, "ln_mod", 1);
    if (M) CK(ln_modulate(A.x.as<float>(), M, D, w.mod + 0 * D, A.e.as<float>() + 0 * D, w.mod + 1 * D,
                          A.e.as<float>() + 1 * D, 6 * D, A.row_req.as<int>(), eps, A.a.as<bf16>(), strm(c)));
  }
  EpiParams eq = epi(A.qkv.p, 3 * D, w.b_qkv);
  const bool ssq = qk_uses_ssq(D);
  if (ssq) {  // the qk-RMSNorm sums come out of the QKV GEMM epilogue
    eq.ssq = A.ssq.as<float>();
    eq.ssq_cols = 2 * D;
  }
  RET(gemm(c, "gemm_qkv", EPI_BF16, M, 3 * D, D, A.a.p, w.w_qkv, eq));
  {
    Scope sc(c, "qk_norm_rope", 1);
    RopeParams rp{A.row_req.as<int>(), A.row_tok.as<int>(), A.req_grid.as<int>(), P.m->cs_tab, P.m->slot_axis,
                  P.m->p_max};
    PackParams pk{};
    if (P.nchunks() > kMaxChunks) return fail(c, GS_EUNSUPPORTED, "%d pack chunks (> %d)", P.nchunks(), kMaxChunks);
    pk.ndest = P.nchunks();
    pk.rows = M;
    for (int j = 0; j <= P.nchunks(); ++j) pk.head_off[j] = P.hoff[j];
    for (int j = 0; j < P.nchunks(); ++j) pk.dest_off[j] = static_cast<long long>(M) * P.hoff[j] * P.hd;
    if (P.peer) {  // fused seq->head exchange: chunk j straight into position j's RECV buffers
      std::vector<long long> rd, ob;
      std::vector<int> ol;
      if (!peer_tables(P, i, rd, ol, ob)) return fail(c, GS_ESTATE, "peer tables for a batch with p !| H");
      pk.peer = 1;
      for (int j = 0; j < P.p; ++j) {
        pk.dst_q[j] = P.qr_of[j];
        pk.dst_k[j] = P.kr_of[j];
        pk.dst_v[j] = P.vr_of[j];
      }
      pk.nseq = P.B;
      for (int r = 0; r < P.B; ++r) {
        pk.row_delta[r] = rd[r];
        pk.seq_lo[r] = P.loff[i][r];
      }
    }
    // SP = 1: no exchange, so V is not copied -- the attention reads it in place from the QKV output
    if (M) CK(qk_norm_rope_pack(A.qkv.as<bf16>(), M, D, P.H, w.g_q, w.g_k, eps, rp, pk, A.qs.as<bf16>(),
                                A.ks.as<bf16>(), P.p == 1 ? nullptr : A.vs.as<bf16>(), strm(c),
                                ssq ? A.ssq.as<float>() : nullptr));
  }
  return GS_OK;
}

int block_attn(gs_ctx* c, const Plan& P, int j, RankArena& A) {
  Scope sc(c, "attention", 1);
  std::vector<int> so(P.B), sl(P.B);
  for (int r = 0; r < P.B; ++r) {
    so[r] = P.off_full[r];
    sl[r] = P.reqs[r]->n;
  }
  if (P.p == 1) {
    const int rs = P.H * P.hd;  // V in place: columns [2D, 3D) of the QKV GEMM output (row stride 3D)
    CK(attention_tc(A.qs.p, A.ks.p, A.qkv.as<bf16>() + 2 * rs, A.o.p, P.H, P.hd, rs, rs, rs, so.data(), sl.data(),
                    P.B, c->num_sms, strm(c), nullptr, 3 * rs));
    return GS_OK;
  }
  if (P.peer) {  // fused head->seq exchange: output rows straight into their owners' ORECV
    std::vector<long long> rd, ob;
    std::vector<int> ol;
    if (!peer_tables(P, j, rd, ol, ob)) return fail(c, GS_ESTATE, "peer tables for a batch with p !| H");
    OScatter osc{};
    osc.nown = P.p;
    for (int r = 0; r < P.B; ++r)
      for (int i = 0; i < P.p; ++i) {
        osc.lo[r][i] = ol[static_cast<size_t>(r) * P.p + i];
        osc.base[r][i] = P.orecv_of[i] + ob[static_cast<size_t>(r) * P.p + i];
      }
    const int rs = P.Hf * P.hd;
    CK(attention_tc(A.qr.p, A.kr.p, A.vr.p, nullptr, P.Hf, P.hd, rs, rs, P.D, so.data(), sl.data(), P.B,
                    c->num_sms, strm(c), &osc));
    return GS_OK;
  }
  // full heads of this position
  if (P.Hf) {
    const int rs = P.Hf * P.hd;
    CK(attention_tc(A.qr.p, A.kr.p, A.vr.p, A.o.p, P.Hf, P.hd, rs, rs, rs, so.data(), sl.data(), P.B, c->num_sms,
                    strm(c)));
  }
  // partial-head units: the unit's query chunk of every request against the head's full K / V
  for (size_t t = 0; t < P.units_of[j].size(); ++t) {
    const Unit& u = P.units[P.units_of[j][t]];
    std::vector<int> qo(P.B), ql(P.B);
    for (int r = 0; r < P.B; ++r) {
      qo[r] = P.qpre(r, u.ci);
      ql[r] = P.chunk_hi(r, u.ci) - P.chunk_lo(r, u.ci);
    }
    const bf16* q = A.qr.as<bf16>() + P.unit_q_off(j, static_cast<int>(t));
    const bf16* k = A.kr.as<bf16>() + P.unit_kv_off(j, static_cast<int>(t));
    const bf16* v = A.vr.as<bf16>() + P.unit_kv_off(j, static_cast<int>(t));
    bf16* o = A.o.as<bf16>() + P.unit_q_off(j, static_cast<int>(t));
    CK(attention_tc_segments(q, k, v, o, 1, P.hd, P.hd, P.hd, P.hd, qo.data(), ql.data(), so.data(), sl.data(), P.B,
                             strm(c)));
  }
  return GS_OK;
}

// Text cross-attention (NEXT-1, reading 19): x += CrossAttn(LN_aff(x), context) W_co^T +
// b_co.  Token-local: each rank's query rows attend to the request's replicated context K/V, so
// no SP exchange is needed.
int block_cross(gs_ctx* c, const Plan& P, int i, RankArena& A, int l) {
  const int M = P.rows[i], D = P.D, Lt = P.m->desc.text_len, NL = P.m->desc.layers;
  const BlockW& w = P.m->blocks[l];
  const float eps = P.m->desc.eps;
  if (!M) return GS_OK;
  {
    Scope sc(c, "ln_mod", 1);
    CK(ln_modulate(A.x.as<float>(), M, D, w.ln3_shift, P.m->zeros, w.ln3_scale_m1, P.m->zeros, 0,
                   A.row_req.as<int>(), eps, A.a.as<bf16>(), strm(c)));
  }
  RET(gemm(c, "gemm_cross_q", EPI_BF16, M, D, D, A.a.p, w.w_cq, epi(A.qc.p, D, w.b_cq)));
  {
    Scope sc(c, "rmsnorm", 1);
    CK(rmsnorm_rows(A.qc.as<bf16>(), D, M, D, w.g_cq, eps, A.qc.as<bf16>(), strm(c)));
  }
  const int li = local_index(c, P.ranks[i]);
  for (int v = 0; v < P.B; ++v) {
    const int cnt = P.hi[i][v] - P.lo[i][v];
    if (!cnt) continue;
    Scope sc(c, "attention_cross", 1);
    const size_t per = static_cast<size_t>(Lt) * D;
    const bf16* kv = P.reqs[v]->ctx_kv.at(li).as<bf16>() + (static_cast<size_t>(P.branch[v]) * NL + l) * 2 * per;
    bf16* q = A.qc.as<bf16>() + static_cast<size_t>(P.loff[i][v]) * D;
    const int zero = 0;
    // in place: each CTA reads its Q tiles before it writes the same rows / head columns of O
    CK(attention_tc_segments(q, kv, kv + per, q, P.H, P.hd, D, D, D, &zero, &cnt, &zero, &Lt, 1, strm(c)));
  }
  RET(gemm(c, "gemm_cross_o", EPI_ADD_F32, M, D, D, A.qc.p, w.w_co, epi(A.x.p, D, w.b_co)));
  return GS_OK;
}

int block_post(gs_ctx* c, const Plan& P, int i, RankArena& A, int l) {
  const int M = P.rows[i], D = P.D, F = P.F;
  const BlockW& w = P.m->blocks[l];
  EpiParams eo = epi(A.x.p, D, w.b_o);
  eo.gate_a = w.mod + 2 * D;
  eo.gate_b = A.e.as<float>() + 2 * D;
  eo.gate_b_stride = 6 * D;
  eo.row_req = A.row_req.as<int>();
  const void* oin = P.p == 1 ? A.o.p : A.orecv.p;
  RET(gemm(c, "gemm_o", EPI_RESID_F32, M, D, D, oin, w.w_o, eo));
  if (P.text) RET(block_cross(c, P, i, A, l));
  {
    Scope sc(c, "ln_mod", 1);
    if (M) CK(ln_modulate(A.x.as<float>(), M, D, w.mod + 3 * D, A.e.as<float>() + 3 * D, w.mod + 4 * D,
                          A.e.as<float>() + 4 * D, 6 * D, A.row_req.as<int>(), P.m->desc.eps, A.a.as<bf16>(),
                          strm(c)));
  }
  RET(gemm(c, "gemm_mlp_up", EPI_GELU_BF16, M, F, D, A.a.p, w.w_1, epi(A.h.p, F, w.b_1)));
  EpiParams e2 = epi(A.x.p, D, w.b_2);
  e2.gate_a = w.mod + 5 * D;
  e2.gate_b = A.e.as<float>() + 5 * D;
  e2.gate_b_stride = 6 * D;
  e2.row_req = A.row_req.as<int>();
  RET(gemm(c, "gemm_mlp_down", EPI_RESID_F32, M, D, F, A.h.p, w.w_2, e2));
  return GS_OK;
}

int step_prologue(gs_ctx* c, const Plan& P, int i, RankArena& A, const float* t) {
  const int M = P.rows[i], D = P.D;
  Model* m = P.m;
  {
    Scope sc(c, "time_embed", 4);
    TimeEmbedW tw{m->w_t1, m->b_t1, m->w_t2, m->b_t2, m->w_tp, m->b_tp, D, m->desc.freq_dim};
    CK(time_embed(tw, static_cast<int>(P.ureqs.size()), t, A.temb.as<float>(), A.e0.as<float>(),
                  A.e.as<float>(), strm(c)));
  }
  {
    Scope sc(c, "patch_embed", 1);
    if (M) CK(f32_to_bf16(A.zpack.as<float>(), A.zb.as<bf16>(), static_cast<long long>(M) * m->desc.lat, strm(c)));
  }
  RET(gemm(c, "patch_embed", EPI_F32, M, D, m->desc.lat, A.zb.p, m->w_pe, epi(A.x.p, D, m->b_pe)));
  return GS_OK;
}

int step_epilogue(gs_ctx* c, const Plan& P, int i, RankArena& A, const float* dsig) {
  const int M = P.rows[i], D = P.D;
  Model* m = P.m;
  {
    Scope sc(c, "head", 1);
    if (M) CK(ln_modulate(A.x.as<float>(), M, D, m->mod_head, A.e0.as<float>(), m->mod_head + D, A.e0.as<float>(), D,
                          A.row_req.as<int>(), m->desc.eps, A.a.as<bf16>(), strm(c)));
  }
  if (!P.text) {
    EpiParams eh = epi(A.zpack.p, m->desc.lat, m->b_head);
    eh.row_req = A.row_req.as<int>();
    for (size_t r = 0; r < P.ureqs.size(); ++r) eh.dsig[r] = dsig[r];
    RET(gemm(c, "head", EPI_EULER_F32, M, m->desc.lat, D, A.a.p, m->w_head, eh));
    return GS_OK;
  }
  // velocity of every sequence, then classifier-free guidance + Euler on the cond rows
  RET(gemm(c, "head", EPI_F32, M, m->desc.lat, D, A.a.p, m->w_head, epi(A.vbuf.p, m->desc.lat, m->b_head)));
  const size_t lat = m->desc.lat;
  for (int v = 0; v < P.B; ++v) {
    if (P.branch[v] != 0) continue;
    const long long cnt = static_cast<long long>(P.hi[i][v] - P.lo[i][v]) * lat;
    if (!cnt) continue;
    const float* vu = nullptr;
    float* zu = nullptr;  // the uncond rows hold a copy of the latent: keep it current across steps
    for (int u = 0; u < P.B; ++u)
      if (P.real[u] == P.real[v] && P.branch[u] == 1) {
        vu = A.vbuf.as<float>() + static_cast<size_t>(P.loff[i][u]) * lat;
        zu = A.zpack.as<float>() + static_cast<size_t>(P.loff[i][u]) * lat;
      }
    Scope sc(c, "cfg_euler", 1);
    const size_t off = static_cast<size_t>(P.loff[i][v]) * lat;
    CK(cfg_euler(A.zpack.as<float>() + off, zu, A.vbuf.as<float>() + off, vu, cnt, dsig[P.real[v]], P.reqs[v]->cfg,
                 strm(c)));
  }
  return GS_OK;
}

// Positions of the plan owned by this process.
std::vector<int> local_positions(gs_ctx* c, const Plan& P) {
  std::vector<int> out;
  for (int i = 0; i < P.p; ++i)
    if (local_index(c, P.ranks[i]) >= 0) out.push_back(i);
  return out;
}

int run_one_step(gs_ctx* c, const Plan& P, const std::vector<int>& mine) {
  float t[MAX_BATCH], dsig[MAX_BATCH];
  for (size_t r = 0; r < P.ureqs.size(); ++r) {
    const Request* q = P.ureqs[r];
    const double s0 = sigma_at(q->step_idx, q->steps, P.m->desc.flow_shift);
    const double s1 = sigma_at(q->step_idx + 1, q->steps, P.m->desc.flow_shift);
    t[r] = static_cast<float>(1000.0 * s0);
    dsig[r] = static_cast<float>(s1 - s0);
  }
  for (int i : mine) RET(step_prologue(c, P, i, c->local[local_index(c, P.ranks[i])], t));
  for (int l = 0; l < P.m->desc.layers; ++l) {
    for (int i : mine) RET(block_pre(c, P, i, c->local[local_index(c, P.ranks[i])], l));
    if (P.p > 1) RET(P.peer ? peer_barrier(c, P, mine) : exchange_qkv(c, P));
    for (int i : mine) RET(block_attn(c, P, i, c->local[local_index(c, P.ranks[i])]));
    if (P.p > 1) RET(P.peer ? peer_barrier(c, P, mine) : exchange_o(c, P));
    for (int i : mine) RET(block_post(c, P, i, c->local[local_index(c, P.ranks[i])], l));
  }
  for (int i : mine) RET(step_epilogue(c, P, i, c->local[local_index(c, P.ranks[i])], dsig));
  return GS_OK;
}

// Agree on "stop at this boundary" across the SP group (NCCL mode): OR of local flags.  The same
// exchange carries each position's arena generation (gens[j] for SP position j; may be null), which
// lets the first step of a run re-use cached IPC mappings (peer_setup).
int agree_stop(gs_ctx* c, const Plan& P, int local_flag, int* stop, unsigned* gens = nullptr) {
  if (c->emulated || P.p == 1) {
    *stop = local_flag;
    return GS_OK;
  }
  const int me = my_position(c, P);
  if (me < 0) return fail(c, GS_ESTATE, "agree_stop: this process is not in the SP group");
  c->h_flag[0] = local_flag;
  c->h_flag[1] = static_cast<int>(c->arena_gen);
  CK(cudaMemcpyAsync(c->d_flag, c->h_flag, 8, cudaMemcpyHostToDevice, strm(c)));
  NK(ncclGroupStart());
  for (int j = 0; j < P.p; ++j) {
    if (j == me) continue;
    NK(ncclSend(c->d_flag, 2, ncclInt32, P.ranks[j], c->comm, strm(c)));
    NK(ncclRecv(c->d_flag + 2 + 2 * j, 2, ncclInt32, P.ranks[j], c->comm, strm(c)));
  }
  NK(ncclGroupEnd());
  CK(cudaMemcpyAsync(c->h_flag + 2, c->d_flag + 2, 16 * 4, cudaMemcpyDeviceToHost, strm(c)));
  CK(cudaStreamSynchronize(strm(c)));
  int s = local_flag;
  for (int j = 0; j < P.p; ++j) {
    if (j == me) continue;
    s |= c->h_flag[2 + 2 * j];
    if (gens) gens[j] = static_cast<unsigned>(c->h_flag[3 + 2 * j]);
  }
  if (gens) gens[me] = c->arena_gen;
  *stop = s;
  return GS_OK;
}

Request* find_req(gs_ctx* c, gs_req id) {
  std::lock_guard<std::mutex> g(c->table_mu);
  auto it = c->reqs.find(id);
  return it == c->reqs.end() ? nullptr : it->second.get();
}

int alloc_shard(gs_ctx* c, Shard& s, int lat) {
  s.bytes = static_cast<size_t>(std::max(s.hi - s.lo, 1)) * lat * 4;
  s.z = static_cast<float*>(pool_alloc(c, s.bytes));
  if (!s.z) return fail(c, GS_ENOMEM, "latent shard alloc failed");
  return GS_OK;
}

// Context K / V of every layer for a request on local rank li (replicated on every rank of its
// placement, built on first use there): c = W_te2 GELU(W_te1 emb + b) + b (bf16), then per layer
// [k|v] = c W_ckv^T + b_ckv, k <- RMSNorm(k) g_ck.  Layout [nb][layers][2][text_len][D] bf16.
int ensure_text_cache(gs_ctx* c, Model* m, Request* q, int li) {
  if (!m->desc.cross_attn) return GS_OK;
  DevBuf& buf = q->ctx_kv[li];
  if (buf.p) return GS_OK;
  const int Lt = m->desc.text_len, T = m->desc.text_dim, D = m->desc.dim, NL = m->desc.layers, nb = q->nb;
  const size_t per = static_cast<size_t>(Lt) * D;
  buf.cap = static_cast<size_t>(nb) * NL * 2 * per * 2;
  buf.p = pool_alloc(c, buf.cap);
  if (!buf.p) return fail(c, GS_ENOMEM, "text cache alloc failed");
  DevBuf emb, h1, cx, kv;
  auto cleanup = [&] {
    cudaStreamSynchronize(strm(c));
    for (DevBuf* b : {&emb, &h1, &cx, &kv})
      if (b->p) cudaFree(b->p);
  };
  int rc = GS_OK;
  do {
    const size_t rows = static_cast<size_t>(nb) * Lt;
    if ((rc = ensure(c, emb, rows * T * 2)) != GS_OK) break;
    if ((rc = ensure(c, h1, rows * D * 2)) != GS_OK) break;
    if ((rc = ensure(c, cx, rows * D * 2)) != GS_OK) break;
    if ((rc = ensure(c, kv, rows * 2 * D * 2)) != GS_OK) break;
    cudaError_t e = cudaSuccess;
    if (!q->prompt_host.empty())
      e = cudaMemcpyAsync(emb.p, q->prompt_host.data(), rows * T * 2, cudaMemcpyHostToDevice, strm(c));
    else
      for (int b = 0; b < nb && e == cudaSuccess; ++b)
        e = rng_normal_bf16(emb.as<bf16>() + static_cast<size_t>(b) * Lt * T, static_cast<long long>(Lt) * T,
                            q->prompt_seed, 50 + b, strm(c));
    if (e != cudaSuccess) {
      rc = fail(c, GS_ECUDA, "prompt upload: %s", cudaGetErrorString(e));
      break;
    }
    if ((rc = gemm(c, "text_embed", EPI_GELU_BF16, rows, D, T, emb.p, m->w_te1, epi(h1.p, D, m->b_te1))) != GS_OK) break;
    if ((rc = gemm(c, "text_embed", EPI_BF16, rows, D, D, h1.p, m->w_te2, epi(cx.p, D, m->b_te2))) != GS_OK) break;
    for (int l = 0; l < NL && rc == GS_OK; ++l) {
      const BlockW& w = m->blocks[l];
      if ((rc = gemm(c, "text_kv", EPI_BF16, rows, 2 * D, D, cx.p, w.w_ckv, epi(kv.p, 2 * D, w.b_ckv))) != GS_OK) break;
      for (int b = 0; b < nb && rc == GS_OK; ++b) {
        bf16* dst = buf.as<bf16>() + (static_cast<size_t>(b) * NL + l) * 2 * per;
        const bf16* src = kv.as<bf16>() + static_cast<size_t>(b) * Lt * 2 * D;
        e = rmsnorm_rows(src, 2 * D, Lt, D, w.g_ck, m->desc.eps, dst, strm(c));
        if (e == cudaSuccess)
          e = cudaMemcpy2DAsync(dst + per, D * 2, src + D, 2 * D * 2, D * 2, Lt, cudaMemcpyDeviceToDevice, strm(c));
        if (e != cudaSuccess) rc = fail(c, GS_ECUDA, "text cache: %s", cudaGetErrorString(e));
      }
    }
  } while (0);
  cleanup();
  if (rc != GS_OK && buf.p) {
    pool_free(c, buf.p, buf.cap);
    buf.p = nullptr;
    buf.cap = 0;
  }
  return rc;
}

void free_text_cache(gs_ctx* c, Request* q) {
  for (auto& kv : q->ctx_kv) pool_free(c, kv.second.p, kv.second.cap);
  q->ctx_kv.clear();
}

void free_shards(gs_ctx* c, std::vector<Shard>& v) {
  for (Shard& s : v) {
    pool_free(c, s.z, s.bytes);
    s.z = nullptr;
  }
}

}  // namespace

// ==================================================================== C-ABI
extern "C" {

int gs_nccl_unique_id(void* out128) {
  if (!out128) return GS_EINVAL;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return GS_ENCCL;
  memcpy(out128, &id, sizeof(id));
  return GS_OK;
}

// nlanes: one stream per local rank (lane 0 = the caller thread's stream); per global rank an idle
// busy slot; the peer-store barrier words (fused all-to-alls, p > 1 only).
static int init_common(gs_ctx* c, int device, int nlanes) {
  DBG("init: device %d lanes %d", device, nlanes);
  CK(cudaSetDevice(device));
  CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
  CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  c->lanes.push_back(c->stream);
  for (int i = 1; i < nlanes; ++i) {
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    c->lanes.push_back(s);
  }
  c->busy.assign(c->world, 0);
  CK(cudaMallocHost(&c->h_flag, 64 * 4));
  CK(cudaMalloc(&c->d_flag, 64 * 4));
  CK(cudaMallocHost(&c->h_id, 4 * 8));
  CK(cudaMalloc(&c->d_id, 4 * 8));
  if (c->world > 1) {
    // words [0, 8): barrier counters per source rank, [8, 16): mapping-probe counters
    const size_t words = static_cast<size_t>(c->emulated ? c->world : 1) * 16;
    CK(cudaMalloc(&c->flags, words * 8));
    CK(cudaMemset(c->flags, 0, words * 8));
  }
  DBG("init: done");
  return GS_OK;
}

int gs_init(int device, int world_size, int rank, const void* nccl_uid, gs_ctx** out) {
  if (!out || world_size < 1 || rank < 0 || rank >= world_size) return GS_EINVAL;
  gs_ctx* c = new gs_ctx();
  c->device = device;
  c->world = world_size;
  c->my_rank = rank;
  int rc = init_common(c, device, 1);
  if (rc != GS_OK) {
    *out = c;
    return rc;
  }
  c->local.resize(1);
  c->local[0].rank = rank;
  if (world_size > 1) {
    if (!nccl_uid) {
      *out = c;
      return fail(c, GS_EINVAL, "world_size > 1 needs an NCCL unique id");
    }
    ncclUniqueId id;
    memcpy(&id, nccl_uid, sizeof(id));
    ncclResult_t r = ncclCommInitRank(&c->comm, world_size, id, rank);
    if (r == ncclSuccess) r = ncclCommSplit(c->comm, 0, rank, &c->ctrl, nullptr);
    if (r != ncclSuccess) {
      *out = c;
      return fail(c, GS_ENCCL, "ncclCommInitRank / ncclCommSplit: %s", ncclGetErrorString(r));
    }
    // Programmatic dependent launch stays on: only OUR kernels carry the PDL launch attribute, so
    // (a) an NCCL kernel enqueued after one of ours is a plain launch and waits for its completion,
    // and (b) one of ours enqueued after an NCCL kernel may only start early if that kernel triggers
    // griddepcontrol.launch_dependents, which NCCL's kernels do not -- the trigger is then implicit at
    // their completion.  The fused peer-store exchange has no NCCL kernels on the data path at all.
    // (Unmeasured on two physical GPUs: gpurun gives one; tests/test_gpu_multiproc.py covers it.)
  }
  *out = c;
  return GS_OK;
}

int gs_init_emulated(int device, int world_size, gs_ctx** out) {
  if (!out || world_size < 1 || world_size > 8) return GS_EINVAL;
  gs_ctx* c = new gs_ctx();
  c->device = device;
  c->world = world_size;
  c->emulated = true;
  int rc = init_common(c, device, world_size);
  c->local.resize(world_size);
  for (int r = 0; r < world_size; ++r) c->local[r].rank = r;
  *out = c;
  return rc;
}

void gs_destroy(gs_ctx* c) {
  if (!c) return;
  {
    std::vector<gs_ticket> open;
    {
      std::lock_guard<std::mutex> g(c->table_mu);
      for (auto& kv : c->tickets) open.push_back(kv.first);
    }
    for (gs_ticket t : open) gs_wait(c, t, nullptr);
  }
  cudaSetDevice(c->device);
  for (size_t i = 1; i < c->lanes.size(); ++i) cudaStreamSynchronize(c->lanes[i]);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto& kv : c->reqs) {
    free_shards(c, kv.second->shards);
    free_text_cache(c, kv.second.get());
  }
  for (auto& kv : c->pool) cudaFree(kv.second);
  c->pool.clear();
  for (auto& m : c->models)
    for (void* p : m->allocs) cudaFree(p);
  for (auto& v : c->vaes) {
    for (void* p : v->allocs) cudaFree(p);
    for (DevBuf* b : {&v->act[0], &v->act[1], &v->act[2], &v->act[3], &v->lat_stage, &v->vid_stage})
      if (b->p) cudaFree(b->p);
  }
  for (auto& A : c->local) {
    DevBuf* bufs[] = {&A.x, &A.a, &A.qkv, &A.qs, &A.ks, &A.vs, &A.qr, &A.kr, &A.vr, &A.o, &A.orecv,
                      &A.ostage, &A.h, &A.zpack, &A.zb, &A.e0, &A.e, &A.temb, &A.row_req, &A.row_tok,
                      &A.req_grid, &A.qc, &A.vbuf, &A.ssq};
    for (DevBuf* b : bufs)
      if (b->p) cudaFree(b->p);
  }
  for (auto& pm : c->peers)
    for (void* p : pm.p)
      if (p) cudaIpcCloseMemHandle(p);
  if (c->flags) cudaFree(c->flags);
  if (c->ipc_dev) cudaFree(c->ipc_dev);
  for (auto e : c->event_pool) cudaEventDestroy(e);
  if (c->ev_order) cudaEventDestroy(c->ev_order);
  if (c->ctrl) ncclCommDestroy(c->ctrl);
  if (c->comm) ncclCommDestroy(c->comm);
  if (c->h_flag) cudaFreeHost(c->h_flag);
  if (c->d_flag) cudaFree(c->d_flag);
  if (c->h_id) cudaFreeHost(c->h_id);
  if (c->d_id) cudaFree(c->d_id);
  for (size_t i = 1; i < c->lanes.size(); ++i) cudaStreamDestroy(c->lanes[i]);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

const char* gs_last_error(gs_ctx* c) { return c ? c->err.c_str() : "null context"; }

int gs_set_option(gs_ctx* c, const char* key, long long value) {
  if (!c || !key) return GS_EINVAL;
  if (strcmp(key, "a2a") == 0) {
    if (value != 0 && value != 1) return fail(c, GS_EINVAL, "a2a option %lld (0 = transfer plans, 1 = peer stores)", value);
    c->a2a_mode = static_cast<int>(value);
    return GS_OK;
  }
  if (strcmp(key, "usp_ring") == 0) {
    if (value != 1 && value != 2 && value != 4 && value != 8)
      return fail(c, GS_EINVAL, "usp_ring %lld (1 = Ulysses only, 2 / 4 / 8 = ring degree)", value);
    c->usp_ring = static_cast<int>(value);
    return GS_OK;
  }
  if (strcmp(key, "gemm_bn") == 0) {
    if (value != 0 && value != 192 && value != 256) return fail(c, GS_EINVAL, "gemm_bn %lld (0, 192, 256)", value);
    g_gemm_bn_override.store(static_cast<int>(value));
    return GS_OK;
  }
  if (strcmp(key, "pdl") == 0) {
    if (value != 0 && value != 1) return fail(c, GS_EINVAL, "pdl %lld (0, 1)", value);
    g_pdl.store(static_cast<int>(value));
    return GS_OK;
  }
  return fail(c, GS_EINVAL, "unknown option '%s'", key);
}

int gs_info(gs_ctx* c, int* num_sms, int* world_size, int* nlocal) {
  if (!c) return GS_EINVAL;
  if (num_sms) *num_sms = c->num_sms;
  if (world_size) *world_size = c->world;
  if (nlocal) *nlocal = static_cast<int>(c->local.size());
  return GS_OK;
}

int gs_model_create(gs_ctx* c, const gs_model_desc* d, int* model_id) {
  if (!c || !d || !model_id) return GS_EINVAL;
  DBG("model_create: enter");
  std::lock_guard<std::mutex> g(c->api_mu);
  DBG("model_create: api_mu");
  RET(no_runs_in_flight(c, "gs_model_create"));
  DBG("model_create: idle checked");
  CK(cudaSetDevice(c->device));
  DBG("model_create: device set, stream %p", (void*)strm(c));
  if (d->dim <= 0 || d->heads <= 0 || d->dim % d->heads || d->dim % 64 || d->dim > 8192 || d->ffn % 256 ||
      d->layers < 1 || d->lat != 64 || d->freq_dim % 2 || d->freq_dim % 64)
    return fail(c, GS_EINVAL, "unsupported model shape (dim %d heads %d ffn %d lat %d)", d->dim, d->heads, d->ffn, d->lat);
  const int hd = d->dim / d->heads;
  if (hd != 64 && hd != 128) return fail(c, GS_EUNSUPPORTED, "head dim %d not in {64, 128}", hd);
  if (d->cross_attn && (d->text_len < 1 || d->text_len > 4096 || d->text_dim < 64 || d->text_dim % 64))
    return fail(c, GS_EINVAL, "bad text shape (len %d dim %d)", d->text_len, d->text_dim);
  auto m = std::make_unique<Model>();
  m->desc = *d;
  m->hd = hd;
  m->blocks.resize(d->layers);
  for (int l = 0; l < d->layers; ++l)
    for (const WSpec& s : all_block_specs(*d)) RET(gen(c, *m, block_slot(m->blocks[l], s.name), s, d->weight_seed + l));
  DBG("model_create: block weights launched");
  for (const WSpec& s : all_global_specs(*d)) RET(gen(c, *m, global_slot(*m, s.name), s, d->weight_seed + 1000000ull));
  if (d->cross_attn) {
    // norm3 affine as ln_modulate tables: LN(x) * (1 + (w - 1)) + b, w - 1 exact in fp32
    const int D = d->dim;
    std::vector<float> zeros(D, 0.f), sm1(D), sh(D);
    std::vector<bf16> wv(D), bv(D);
    void* pz = nullptr;
    CK(cudaMalloc(&pz, D * 4));
    m->allocs.push_back(pz);
    CK(cudaMemcpy(pz, zeros.data(), D * 4, cudaMemcpyHostToDevice));
    m->zeros = static_cast<float*>(pz);
    CK(cudaStreamSynchronize(strm(c)));
    for (int l = 0; l < d->layers; ++l) {
      BlockW& b = m->blocks[l];
      CK(cudaMemcpy(wv.data(), b.ln3_w, D * 2, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(bv.data(), b.ln3_b, D * 2, cudaMemcpyDeviceToHost));
      for (int i = 0; i < D; ++i) {
        sm1[i] = __bfloat162float(wv[i]) - 1.0f;
        sh[i] = __bfloat162float(bv[i]);
      }
      void *ps = nullptr, *pb = nullptr;
      CK(cudaMalloc(&ps, D * 4));
      m->allocs.push_back(ps);
      CK(cudaMalloc(&pb, D * 4));
      m->allocs.push_back(pb);
      CK(cudaMemcpy(ps, sm1.data(), D * 4, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(pb, sh.data(), D * 4, cudaMemcpyHostToDevice));
      b.ln3_scale_m1 = static_cast<float*>(ps);
      b.ln3_shift = static_cast<float*>(pb);
    }
  }
  // RoPE table (reading 1 / SURVEY.md §8(c) step 4): slots [d/2 - 2 floor(d/6), floor(d/6), floor(d/6)]
  const int half = hd / 2, s3 = hd / 6;
  const int slots[3] = {half - 2 * s3, s3, s3};
  std::vector<int> axis(half);
  std::vector<double> freq(half);
  int k = 0;
  for (int a = 0; a < 3; ++a)
    for (int j = 0; j < slots[a]; ++j, ++k) {
      axis[k] = a;
      freq[k] = std::pow(static_cast<double>(d->rope_theta), -2.0 * j / (2.0 * slots[a]));
    }
  std::vector<float2> tab(static_cast<size_t>(m->p_max) * half);
  for (int p = 0; p < m->p_max; ++p)
    for (int s = 0; s < half; ++s) {
      const double ang = p * freq[s];
      tab[static_cast<size_t>(p) * half + s] = make_float2(static_cast<float>(std::cos(ang)), static_cast<float>(std::sin(ang)));
    }
  void *pt = nullptr, *pa = nullptr;
  CK(cudaMalloc(&pt, tab.size() * sizeof(float2)));
  m->allocs.push_back(pt);
  CK(cudaMalloc(&pa, axis.size() * 4));
  m->allocs.push_back(pa);
  CK(cudaMemcpy(pt, tab.data(), tab.size() * sizeof(float2), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(pa, axis.data(), axis.size() * 4, cudaMemcpyHostToDevice));
  m->cs_tab = static_cast<float2*>(pt);
  m->slot_axis = static_cast<int*>(pa);
  DBG("model_create: syncing");
  CK(cudaStreamSynchronize(strm(c)));
  DBG("model_create: synced");
  c->models.push_back(std::move(m));
  *model_id = static_cast<int>(c->models.size()) - 1;
  return GS_OK;
}

int gs_get_weight(gs_ctx* c, int model, int layer, const char* name, void* host, size_t bytes) {
  if (!c || !name || !host) return GS_EINVAL;
  if (model < 0 || model >= static_cast<int>(c->models.size())) return fail(c, GS_EINVAL, "bad model id");
  Model& m = *c->models[model];
  const auto specs = layer < 0 ? all_global_specs(m.desc) : all_block_specs(m.desc);
  if (layer >= m.desc.layers) return fail(c, GS_EINVAL, "bad layer");
  for (const WSpec& s : specs) {
    if (strcmp(s.name, name)) continue;
    const size_t want = s.rows * s.cols * (s.kind == RNG_F32_SCALED ? 4 : 2);
    if (bytes != want) return fail(c, GS_EINVAL, "%s is %zu bytes, got %zu", name, want, bytes);
    void** slot = layer < 0 ? global_slot(m, name) : block_slot(m.blocks[layer], name);
    CK(cudaSetDevice(c->device));
    CK(cudaStreamSynchronize(strm(c)));
    CK(cudaMemcpy(host, *slot, bytes, cudaMemcpyDeviceToHost));
    return GS_OK;
  }
  return fail(c, GS_EINVAL, "unknown tensor %s", name);
}

}  // extern "C"

// ------------------------------------------------------------------ requests and runs
namespace {

// Sets this thread's launch stream to the lane of `rank` for the guard's lifetime (emulated mode:
// one lane per virtual rank, so disjoint SP groups run on different streams; NCCL mode: lane 0).
struct LaneGuard {
  cudaStream_t saved;
  LaneGuard(gs_ctx* c, int rank) : saved(tl_stream) {
    const int li = local_index(c, rank);
    tl_stream = c->lanes[li >= 0 && li < static_cast<int>(c->lanes.size()) ? li : 0];
  }
  ~LaneGuard() { tl_stream = saved; }
};

// GS_ESTATE if a rank of `ranks` belongs to an in-flight run (caller holds table_mu).
int check_idle(gs_ctx* c, const int* ranks, int n, const char* what) {
  for (int i = 0; i < n; ++i)
    if (c->busy[ranks[i]])
      return fail(c, GS_ESTATE, "%s: rank %d belongs to in-flight run %llu (GPU sets of concurrent runs must be "
                  "disjoint)", what, ranks[i], (unsigned long long)c->busy[ranks[i]]);
  return GS_OK;
}

int no_runs_in_flight(gs_ctx* c, const char* what) {
  std::lock_guard<std::mutex> g(c->table_mu);
  if (!c->tickets.empty()) return fail(c, GS_ESTATE, "%s needs every run waited for (%zu in flight)", what, c->tickets.size());
  return GS_OK;
}

// Allocate and initialise the latent shards of q on `ranks` (z_T from its seed or host copy).
int place_shards(gs_ctx* c, Request* q, const int* ranks, int nranks) {
  const int lat = c->models[q->model]->desc.lat;
  LaneGuard lane(c, ranks[0]);
  std::vector<Shard> sh(nranks);
  int rc = GS_OK;
  for (int i = 0; i < nranks && rc == GS_OK; ++i) {
    Shard& s = sh[i];
    s.rank = ranks[i];
    shard_bounds(q->n, nranks, i, &s.lo, &s.hi);
    if (local_index(c, s.rank) < 0) continue;
    if ((rc = alloc_shard(c, s, lat)) != GS_OK) break;
    cudaError_t e;
    if (!q->init_host.empty())
      e = cudaMemcpyAsync(s.z, q->init_host.data() + static_cast<size_t>(s.lo) * lat,
                          static_cast<size_t>(s.hi - s.lo) * lat * 4, cudaMemcpyHostToDevice, strm(c));
    else
      e = rng_noise(s.z, s.lo, s.hi - s.lo, lat, q->noise_seed, strm(c));
    if (e != cudaSuccess) rc = fail(c, GS_ECUDA, "initial latent: %s", cudaGetErrorString(e));
  }
  cudaError_t e = cudaStreamSynchronize(strm(c));
  if (rc == GS_OK && e != cudaSuccess) rc = fail(c, GS_ECUDA, "initial latent: %s", cudaGetErrorString(e));
  if (rc != GS_OK) {
    free_shards(c, sh);
    return rc;
  }
  q->init_host.clear();
  q->init_host.shrink_to_fit();
  q->shards = std::move(sh);
  q->ranks.assign(ranks, ranks + nranks);
  return GS_OK;
}

// NCCL mode: every process of the job submits every request (gs.h), so the id sequence agrees; a
// min/max all-reduce of the new id over the world detects a process that skipped a submit.
int check_job_wide_id(gs_ctx* c, gs_req id) {
  if (c->emulated || c->world == 1) return GS_OK;
  long long* h = c->h_id;
  long long* d = c->d_id;
  h[0] = static_cast<long long>(id);
  h[1] = -static_cast<long long>(id);
  CK(cudaMemcpyAsync(d, h, 16, cudaMemcpyHostToDevice, strm(c)));
  NK(ncclAllReduce(d, d + 2, 2, ncclInt64, ncclMax, c->ctrl, strm(c)));
  CK(cudaMemcpyAsync(h + 2, d + 2, 16, cudaMemcpyDeviceToHost, strm(c)));
  CK(cudaStreamSynchronize(strm(c)));
  if (h[2] != static_cast<long long>(id) || -h[3] != static_cast<long long>(id))
    return fail(c, GS_ESTATE, "request id %llu differs across processes (ids %lld..%lld): every process must submit "
                "every request", (unsigned long long)id, -h[3], h[2]);
  return GS_OK;
}

}  // namespace

extern "C" {

static int submit_impl(gs_ctx* c, int model, int width, int height, int frames, int steps, uint64_t noise_seed,
                       const float* init_latent, const int* ranks, int nranks, bool text, uint64_t prompt_seed,
                       float cfg_scale, const void* prompt_embeds, gs_req* out) {
  if (!c || !out) return GS_EINVAL;
  std::lock_guard<std::mutex> g(c->api_mu);
  CK(cudaSetDevice(c->device));
  if (model < 0 || model >= static_cast<int>(c->models.size())) return fail(c, GS_EINVAL, "bad model id");
  if (width <= 0 || height <= 0 || width % 16 || height % 16 || frames < 1 || (frames - 1) % 4 || steps < 1)
    return fail(c, GS_EINVAL, "bad request shape %dx%d frames %d steps %d", width, height, frames, steps);
  const bool queued = ranks == nullptr && nranks == 0;
  if (!queued) RET(check_ranks(c, ranks, nranks));
  Model& m = *c->models[model];
  if (text != (m.desc.cross_attn != 0))
    return fail(c, GS_EINVAL, text ? "gs_submit_text needs a cross-attention model"
                                   : "cross-attention model: submit with gs_submit_text");
  auto q = std::make_unique<Request>();
  q->model = model;
  q->grid[0] = 1 + (frames - 1) / 4;
  q->grid[1] = height / 16;
  q->grid[2] = width / 16;
  if (q->grid[0] > m.p_max || q->grid[1] > m.p_max || q->grid[2] > m.p_max)
    return fail(c, GS_EINVAL, "token grid exceeds RoPE table (%d)", m.p_max);
  q->n = q->grid[0] * q->grid[1] * q->grid[2];
  q->steps = steps;
  q->noise_seed = noise_seed;
  if (init_latent) q->init_host.assign(init_latent, init_latent + static_cast<size_t>(q->n) * m.desc.lat);
  if (text) {
    q->nb = cfg_scale > 0.f ? 2 : 1;
    q->cfg = cfg_scale > 0.f ? cfg_scale : 0.f;
    q->prompt_seed = prompt_seed;
    if (prompt_embeds) {
      const size_t n = static_cast<size_t>(q->nb) * m.desc.text_len * m.desc.text_dim;
      q->prompt_host.assign(static_cast<const uint16_t*>(prompt_embeds), static_cast<const uint16_t*>(prompt_embeds) + n);
    }
  }
  {
    std::lock_guard<std::mutex> g2(c->table_mu);
    if (!queued) RET(check_idle(c, ranks, nranks, "gs_submit"));
    q->id = c->next_req++;
  }
  RET(check_job_wide_id(c, q->id));
  if (queued)
    q->state = GS_REQ_QUEUED;
  else
    RET(place_shards(c, q.get(), ranks, nranks));
  std::lock_guard<std::mutex> g2(c->table_mu);
  *out = q->id;
  c->reqs[q->id] = std::move(q);
  return GS_OK;
}

int gs_submit(gs_ctx* c, int model, int width, int height, int frames, int steps, uint64_t noise_seed,
              const float* init_latent, const int* ranks, int nranks, gs_req* out) {
  return submit_impl(c, model, width, height, frames, steps, noise_seed, init_latent, ranks, nranks, false, 0, 0.f,
                     nullptr, out);
}

int gs_submit_text(gs_ctx* c, int model, int width, int height, int frames, int steps, uint64_t noise_seed,
                   uint64_t prompt_seed, float cfg_scale, const float* init_latent, const void* prompt_embeds,
                   const int* ranks, int nranks, gs_req* out) {
  return submit_impl(c, model, width, height, frames, steps, noise_seed, init_latent, ranks, nranks, true,
                     prompt_seed, cfg_scale, prompt_embeds, out);
}

int gs_place(gs_ctx* c, gs_req id, const int* ranks, int nranks) {
  if (!c) return GS_EINVAL;
  std::lock_guard<std::mutex> g(c->api_mu);
  CK(cudaSetDevice(c->device));
  RET(check_ranks(c, ranks, nranks));
  Request* q = nullptr;
  {
    std::lock_guard<std::mutex> g2(c->table_mu);
    auto it = c->reqs.find(id);
    if (it == c->reqs.end()) return fail(c, GS_EINVAL, "unknown request");
    q = it->second.get();
    if (q->state != GS_REQ_QUEUED) return fail(c, GS_ESTATE, "gs_place needs a queued request (state %d)", q->state.load());
    RET(check_idle(c, ranks, nranks, "gs_place"));
  }
  RET(place_shards(c, q, ranks, nranks));
  std::lock_guard<std::mutex> g2(c->table_mu);
  q->state = GS_REQ_PLACED;
  return GS_OK;
}

}  // extern "C"

namespace {

// The body of a run (worker thread of ticket t): rows of the batch on each local position, k steps
// with the preemption check at every step boundary, latent back to the shards, states updated.
void run_body(gs_ctx* c, Ticket* t, std::vector<Request*> reqs, int k) {
  cudaSetDevice(c->device);
  tl_err = &t->err;
  const int* ranks = t->ranks.data();
  const int nranks = static_cast<int>(t->ranks.size());
  LaneGuard lane(c, ranks[0]);
  Model* m = c->models[reqs[0]->model].get();
  Plan P;
  make_plan(P, m, reqs, ranks, nranks, c->usp_ring);
  const std::vector<int> mine = local_positions(c, P);
  int done = 0, rc = GS_OK;
  for (int i : mine) {
    RankArena& A = c->local[local_index(c, P.ranks[i])];
    for (Request* q : reqs)
      if (rc == GS_OK) rc = ensure_text_cache(c, m, q, local_index(c, P.ranks[i]));
    if (rc == GS_OK) rc = prepare_rank(c, P, i, A);
    if (rc == GS_OK) rc = move_latent(c, P, i, A, 0);
  }
  for (int s = 0; s < k && rc == GS_OK; ++s) {
    int flag = 0;
    for (Request* q : reqs) flag |= q->preempt.load();
    int stop = 0;
    unsigned gens[8] = {};
    // the first step's agreement also carries the arena generations, so peer_setup can re-use the
    // IPC mappings of an unchanged SP group without exchanging handles (arenas are sized above)
    if (s == 0 && !c->emulated && P.p > 1 && c->a2a_mode == 1) {
      void* bases[5] = {c->local[0].qr.p, c->local[0].kr.p, c->local[0].vr.p, c->local[0].orecv.p, c->flags};
      if (memcmp(bases, c->exported, sizeof bases) != 0) {
        memcpy(c->exported, bases, sizeof bases);
        ++c->arena_gen;
      }
    }
    rc = agree_stop(c, P, flag, &stop, s == 0 ? gens : nullptr);
    if (rc == GS_OK && s == 0) rc = peer_setup(c, P, c->emulated || P.p == 1 ? nullptr : gens);
    if (rc != GS_OK || stop) break;
    cudaEvent_t s0 = nullptr, s1 = nullptr;
    if (c->prof_steps) {
      std::lock_guard<std::mutex> g(c->prof_mu);
      s0 = get_event(c);
      s1 = get_event(c);
      cudaEventRecord(s0, strm(c));
    }
    rc = run_one_step(c, P, mine);
    if (c->prof_steps) cudaEventRecord(s1, strm(c));
    if (rc != GS_OK) break;
    cudaError_t e = cudaStreamSynchronize(strm(c));
    if (c->prof_steps) {  // whole-step device time (gs_stats "step_ms"): the step-time CV of §8(d)
      float ms = 0;
      cudaEventElapsedTime(&ms, s0, s1);
      std::lock_guard<std::mutex> g(c->prof_mu);
      c->step_ms.push_back(ms);
      c->event_pool.push_back(s0);
      c->event_pool.push_back(s1);
    }
    if (e != cudaSuccess) {
      rc = fail(c, GS_ECUDA, "step failed: %s", cudaGetErrorString(e));
      break;
    }
    prof_flush(c);
    for (Request* q : reqs) ++q->step_idx;
    ++done;
  }
  for (int i : mine) {
    int r2 = move_latent(c, P, i, c->local[local_index(c, P.ranks[i])], 1);
    if (rc == GS_OK) rc = r2;
  }
  cudaError_t e = cudaStreamSynchronize(strm(c));
  if (rc == GS_OK && e != cudaSuccess) rc = fail(c, GS_ECUDA, "%s", cudaGetErrorString(e));
  std::lock_guard<std::mutex> g(c->table_mu);
  for (Request* q : reqs) {
    if (q->preempt.exchange(0))
      q->state = GS_REQ_PAUSED;
    else
      q->state = q->step_idx >= q->steps ? GS_REQ_DONE : GS_REQ_PLACED;
  }
  t->rc = rc;
  t->steps_run = done;
  t->finished.store(1);
  tl_err = nullptr;
}

}  // namespace

extern "C" {

int gs_run_steps_async(gs_ctx* c, const gs_req* ids, int nreq, const int* ranks, int nranks, int k,
                       gs_ticket* ticket) {
  if (!c || !ids || !ticket) return GS_EINVAL;
  *ticket = 0;
  std::lock_guard<std::mutex> g(c->api_mu);
  CK(cudaSetDevice(c->device));
  if (nreq < 1 || nreq > MAX_BATCH) return fail(c, GS_EINVAL, "batch of %d requests (1..%d)", nreq, MAX_BATCH);
  RET(check_ranks(c, ranks, nranks));
  if (!c->emulated) {
    bool member = false;
    for (int i = 0; i < nranks; ++i) member |= ranks[i] == c->my_rank;
    if (!member) return fail(c, GS_ESTATE, "this process (rank %d) owns none of the run's ranks", c->my_rank);
  }
  auto t = std::make_unique<Ticket>();
  t->ranks.assign(ranks, ranks + nranks);
  std::vector<Request*> reqs;
  gs_ticket id;
  {
    // validation and the PLACED -> RUNNING transition are one critical section with gs_preempt
    std::lock_guard<std::mutex> g2(c->table_mu);
    for (int r = 0; r < nreq; ++r) {
      auto it = c->reqs.find(ids[r]);
      if (it == c->reqs.end()) return fail(c, GS_EINVAL, "unknown request %llu", (unsigned long long)ids[r]);
      Request* q = it->second.get();
      for (Request* o : reqs)
        if (o == q) return fail(c, GS_EINVAL, "request listed twice");
      if (q->state != GS_REQ_PLACED)
        return fail(c, GS_ESTATE, "request %llu is not runnable (state %d)", (unsigned long long)q->id, q->state.load());
      if (!reqs.empty() && q->model != reqs[0]->model) return fail(c, GS_ESTATE, "batch mixes models");
      if (static_cast<int>(q->ranks.size()) != nranks || !std::equal(q->ranks.begin(), q->ranks.end(), ranks))
        return fail(c, GS_ESTATE, "request %llu is not placed on the given ranks", (unsigned long long)q->id);
      if (k < 0 || q->step_idx + k > q->steps) return fail(c, GS_EINVAL, "k=%d exceeds remaining steps", k);
      reqs.push_back(q);
    }
    RET(check_idle(c, ranks, nranks, "gs_run_steps"));
    id = c->next_ticket++;
    for (int i = 0; i < nranks; ++i) c->busy[ranks[i]] = id;
    for (Request* q : reqs) q->state = GS_REQ_RUNNING;
  }
  Ticket* tp = t.get();
  {
    std::lock_guard<std::mutex> g2(c->table_mu);
    c->tickets[id] = std::move(t);
  }
  tp->th = std::thread(run_body, c, tp, reqs, k);
  *ticket = id;
  return GS_OK;
}

int gs_wait(gs_ctx* c, gs_ticket id, int* steps_run) {
  if (!c) return GS_EINVAL;
  if (steps_run) *steps_run = 0;
  std::unique_ptr<Ticket> t;
  {
    std::lock_guard<std::mutex> g(c->table_mu);
    auto it = c->tickets.find(id);
    if (it == c->tickets.end()) return fail(c, GS_EINVAL, "unknown ticket %llu", (unsigned long long)id);
    t = std::move(it->second);
    c->tickets.erase(it);
  }
  if (t->th.joinable()) t->th.join();
  {
    std::lock_guard<std::mutex> g(c->table_mu);
    for (int r : t->ranks)
      if (c->busy[r] == id) c->busy[r] = 0;
  }
  if (steps_run) *steps_run = t->steps_run;
  if (t->rc != GS_OK) return fail(c, t->rc, "%s", t->err.c_str());
  return GS_OK;
}

int gs_ticket_done(gs_ctx* c, gs_ticket id) {
  if (!c) return GS_EINVAL;
  std::lock_guard<std::mutex> g(c->table_mu);
  auto it = c->tickets.find(id);
  if (it == c->tickets.end()) return fail(c, GS_EINVAL, "unknown ticket %llu", (unsigned long long)id);
  return it->second->finished.load() ? 1 : 0;
}

int gs_run_steps(gs_ctx* c, const gs_req* ids, int nreq, const int* ranks, int nranks, int k, int* steps_run) {
  if (steps_run) *steps_run = 0;
  gs_ticket t = 0;
  RET(gs_run_steps_async(c, ids, nreq, ranks, nranks, k, &t));
  return gs_wait(c, t, steps_run);
}

int gs_preempt(gs_ctx* c, gs_req id, int* steps_done_out) {
  if (!c) return GS_EINVAL;
  std::lock_guard<std::mutex> g(c->table_mu);
  auto it = c->reqs.find(id);
  if (it == c->reqs.end()) return fail(c, GS_EINVAL, "unknown request");
  Request* q = it->second.get();
  if (q->state == GS_REQ_DONE) return fail(c, GS_ESTATE, "request already finished");
  // a run moves PLACED -> RUNNING and back under table_mu: the flag set here is seen by its next
  // step-boundary check, or the request is paused before any run can claim it
  if (q->state == GS_REQ_RUNNING)
    q->preempt.store(1);
  else if (q->state == GS_REQ_PLACED)
    q->state = GS_REQ_PAUSED;
  if (steps_done_out) *steps_done_out = q->step_idx;
  return GS_OK;
}

int gs_resume(gs_ctx* c, gs_req id, const int* ranks, int nranks) {
  if (!c) return GS_EINVAL;
  std::lock_guard<std::mutex> g(c->api_mu);
  CK(cudaSetDevice(c->device));
  RET(check_ranks(c, ranks, nranks));
  Request* q = nullptr;
  {
    std::lock_guard<std::mutex> g2(c->table_mu);
    auto it = c->reqs.find(id);
    if (it == c->reqs.end()) return fail(c, GS_EINVAL, "unknown request");
    q = it->second.get();
    if (q->state != GS_REQ_PAUSED && q->state != GS_REQ_PLACED)
      return fail(c, GS_ESTATE, "resume needs a paused or placed request (state %d)", q->state.load());
    RET(check_idle(c, ranks, nranks, "gs_resume (new ranks)"));
    // NCCL mode: the re-shard is collective over the old ranks' processes too, and a process must not
    // drive the communicator from two threads -> their ranks must be idle.  Emulated mode: reading
    // the old shards is a device copy that does not disturb another run on those ranks.
    if (!c->emulated) RET(check_idle(c, q->ranks.data(), static_cast<int>(q->ranks.size()), "gs_resume (old ranks)"));
  }
  LaneGuard lane(c, ranks[0]);
  const int lat = c->models[q->model]->desc.lat;
  std::vector<Shard> ns(nranks);
  for (int i = 0; i < nranks; ++i) {
    ns[i].rank = ranks[i];
    shard_bounds(q->n, nranks, i, &ns[i].lo, &ns[i].hi);
    if (local_index(c, ns[i].rank) >= 0) {
      int rc = alloc_shard(c, ns[i], lat);
      if (rc != GS_OK) {
        free_shards(c, ns);
        return rc;
      }
    }
  }
  // interval intersections old x new: pure copies, planned on the host
  std::vector<int> old_ranks(q->ranks);
  auto shard_of = [](std::vector<Shard>& v, int rank) -> float* {
    for (Shard& s : v)
      if (s.rank == rank) return s.z;
    return nullptr;
  };
  if (c->emulated) {
    // every rank is local: pair the n-th send of a with the n-th recv of b
    std::vector<std::vector<gs_xfer>> plans(c->world);
    for (int me = 0; me < c->world; ++me)
      plan_reshard(q->n, lat, old_ranks.data(), static_cast<int>(old_ranks.size()), ranks, nranks, me, plans[me]);
    auto bufs = [&](int rank, int id) -> void* {
      return id == GS_BUF_OLD ? shard_of(q->shards, rank) : shard_of(ns, rank);
    };
    const int rc = run_emulated(c, plans, bufs, 4);
    if (rc != GS_OK) {
      cudaStreamSynchronize(strm(c));
      free_shards(c, ns);
      return rc;
    }
  } else {
    std::vector<gs_xfer> plan;
    plan_reshard(q->n, lat, old_ranks.data(), static_cast<int>(old_ranks.size()), ranks, nranks, c->my_rank, plan);
    float* zo = shard_of(q->shards, c->my_rank);
    float* zn = shard_of(ns, c->my_rank);
    bool any_p2p = false;
    for (const gs_xfer& x : plan) any_p2p |= x.op != GS_XFER_COPY;
    if (any_p2p) {
      NK(ncclGroupStart());
      for (const gs_xfer& x : plan) {
        if (x.op == GS_XFER_SEND)
          NK(ncclSend(zo + x.src_off, x.width * 4, ncclUint8, x.peer, c->comm, strm(c)));
        else if (x.op == GS_XFER_RECV)
          NK(ncclRecv(zn + x.dst_off, x.width * 4, ncclUint8, x.peer, c->comm, strm(c)));
      }
      NK(ncclGroupEnd());
    }
    for (const gs_xfer& x : plan)
      if (x.op == GS_XFER_COPY) RET(copy_block(c, zn + x.dst_off, zo + x.src_off, x, 4));
  }
  CK(cudaStreamSynchronize(strm(c)));
  free_shards(c, q->shards);
  free_text_cache(c, q);  // rebuilt on the new ranks at their first step
  std::lock_guard<std::mutex> g2(c->table_mu);
  q->shards = ns;
  q->ranks.assign(ranks, ranks + nranks);
  q->state = q->step_idx >= q->steps ? GS_REQ_DONE : GS_REQ_PLACED;
  return GS_OK;
}

int gs_query(gs_ctx* c, gs_req id, int* steps_done, int* steps_total, int* nranks, int* ranks_out, int* state,
             int* n_tokens) {
  if (!c) return GS_EINVAL;
  std::lock_guard<std::mutex> g(c->table_mu);
  auto it = c->reqs.find(id);
  if (it == c->reqs.end()) return fail(c, GS_EINVAL, "unknown request");
  Request* q = it->second.get();
  if (steps_done) *steps_done = q->step_idx;
  if (steps_total) *steps_total = q->steps;
  if (nranks) *nranks = static_cast<int>(q->ranks.size());
  if (ranks_out)
    for (size_t i = 0; i < q->ranks.size(); ++i) ranks_out[i] = q->ranks[i];
  if (state) *state = q->state;
  if (n_tokens) *n_tokens = q->n;
  return GS_OK;
}

int gs_read_latent(gs_ctx* c, gs_req id, float* host, size_t nfloats) {
  if (!c || !host) return GS_EINVAL;
  std::lock_guard<std::mutex> g(c->api_mu);
  Request* q = find_req(c, id);
  if (!q) return fail(c, GS_EINVAL, "unknown request");
  if (q->state == GS_REQ_RUNNING) return fail(c, GS_ESTATE, "request is running");
  if (q->state == GS_REQ_QUEUED) return fail(c, GS_ESTATE, "request is queued (not placed)");
  const int lat = c->models[q->model]->desc.lat;
  if (nfloats != static_cast<size_t>(q->n) * lat) return fail(c, GS_EINVAL, "latent has %d x %d floats", q->n, lat);
  CK(cudaSetDevice(c->device));
  LaneGuard lane(c, q->ranks[0]);
  CK(cudaStreamSynchronize(strm(c)));
  for (const Shard& s : q->shards)
    if (s.z && s.hi > s.lo)
      CK(cudaMemcpy(host + static_cast<size_t>(s.lo) * lat, s.z, static_cast<size_t>(s.hi - s.lo) * lat * 4,
                    cudaMemcpyDeviceToHost));
  return GS_OK;
}

int gs_release(gs_ctx* c, gs_req id) {
  if (!c) return GS_EINVAL;
  std::lock_guard<std::mutex> g(c->api_mu);  // no run can claim the request meanwhile
  Request* q = find_req(c, id);
  if (!q) return fail(c, GS_EINVAL, "unknown request");
  if (q->state == GS_REQ_RUNNING) return fail(c, GS_ESTATE, "request is running");
  cudaSetDevice(c->device);
  if (!q->ranks.empty()) {
    LaneGuard lane(c, q->ranks[0]);
    cudaStreamSynchronize(strm(c));
  }
  free_shards(c, q->shards);
  free_text_cache(c, q);
  std::lock_guard<std::mutex> g2(c->table_mu);
  c->reqs.erase(id);
  return GS_OK;
}

int gs_profile(gs_ctx* c, int enable, int reset) {
  if (!c) return GS_EINVAL;
  c->prof = enable == 1;
  c->prof_steps = enable == 1 || enable == 2;
  std::lock_guard<std::mutex> g(c->prof_mu);
  if (reset) {
    c->prof_tab.clear();
    c->step_ms.clear();
    c->launches = 0;
  }
  return GS_OK;
}

int gs_stats(gs_ctx* c, char* json, size_t len) {
  if (!c || !json || len == 0) return GS_EINVAL;
  std::lock_guard<std::mutex> g(c->prof_mu);
  std::string s = "{";
  for (auto& kv : c->prof_tab) {
    char buf[160];
    snprintf(buf, sizeof buf, "\"%s\": {\"ms\": %.6f, \"n\": %lld}, ", kv.first.c_str(), kv.second.ms, kv.second.n);
    s += buf;
  }
  s += "\"step_ms\": [";
  for (size_t i = 0; i < c->step_ms.size(); ++i) {
    char sb[32];
    snprintf(sb, sizeof sb, "%s%.4f", i ? ", " : "", c->step_ms[i]);
    s += sb;
  }
  s += "], ";
  char buf[160];
  snprintf(buf, sizeof buf, "\"a2a_peer\": %lld, \"a2a_plan\": %lld, \"launches\": %lld, \"ipc_exchanges\": %lld}",
           c->a2a_peer.load(), c->a2a_plan.load(), c->launches.load(), c->ipc_exchanges);
  s += buf;
  if (s.size() + 1 > len) return fail(c, GS_EINVAL, "stats buffer too small (%zu)", s.size() + 1);
  memcpy(json, s.c_str(), s.size() + 1);
  return GS_OK;
}

int gs_stream(gs_ctx* c, int rank, void** stream_out) {
  if (!c || !stream_out) return GS_EINVAL;
  if (local_index(c, rank) < 0) return fail(c, GS_EINVAL, "rank %d not owned by this process", rank);
  *stream_out = c->lanes[local_index(c, rank)];
  return GS_OK;
}

// ------------------------------------------------------------------ debug entry points
namespace {
// Caller-owned device buffers are typically produced on the legacy default stream (e.g. by
// torch); order the context's non-blocking stream after that work without a host sync.
int order_after_legacy(gs_ctx* c) {
  if (!c->ev_order) CK(cudaEventCreateWithFlags(&c->ev_order, cudaEventDisableTiming));
  CK(cudaEventRecord(c->ev_order, cudaStreamLegacy));
  CK(cudaStreamWaitEvent(strm(c), c->ev_order, 0));
  return GS_OK;
}
}  // namespace

int gs_debug_gemm(gs_ctx* c, int e, int M, int N, int K, const void* A, const void* W, const void* bias, void* out,
                  const float* gate_a, const float* gate_b, int gate_b_stride, const int* row_req,
                  const float* dsig_host) {
  if (!c) return GS_EINVAL;
  std::lock_guard<std::mutex> g(c->api_mu);
  RET(no_runs_in_flight(c, "gs_debug_gemm"));
  CK(cudaSetDevice(c->device));
  RET(order_after_legacy(c));
  EpiParams ep{};
  ep.out = out;
  ep.ldo = N;
  ep.bias = static_cast<const bf16*>(bias);
  ep.gate_a = gate_a;
  ep.gate_b = gate_b;
  ep.gate_b_stride = gate_b_stride;
  ep.row_req = row_req;
  if (dsig_host)
    for (int i = 0; i < 8; ++i) ep.dsig[i] = dsig_host[i];
  cudaError_t err = gemm_bf16_tc(e, M, N, K, A, K, W, K, ep, c->num_sms, strm(c));
  if (err != cudaSuccess) return fail(c, err == cudaErrorInvalidValue ? GS_EINVAL : GS_ECUDA, "gemm: %s", cudaGetErrorString(err));
  CK(cudaStreamSynchronize(strm(c)));
  return GS_OK;
}

int gs_debug_gemm_ssq(gs_ctx* c, int M, int N, int K, const void* A, const void* W, const void* bias, void* out,
                      float* ssq, int ssq_cols) {
  if (!c || !ssq || ssq_cols <= 0 || ssq_cols % 32 || ssq_cols > N) return GS_EINVAL;
  std::lock_guard<std::mutex> g(c->api_mu);
  RET(no_runs_in_flight(c, "gs_debug_gemm_ssq"));
  CK(cudaSetDevice(c->device));
  RET(order_after_legacy(c));
  EpiParams ep{};
  ep.out = out;
  ep.ldo = N;
  ep.bias = static_cast<const bf16*>(bias);
  ep.ssq = ssq;
  ep.ssq_cols = ssq_cols;
  cudaError_t err = gemm_bf16_tc(EPI_BF16, M, N, K, A, K, W, K, ep, c->num_sms, strm(c));
  if (err != cudaSuccess) return fail(c, err == cudaErrorInvalidValue ? GS_EINVAL : GS_ECUDA, "gemm: %s", cudaGetErrorString(err));
  CK(cudaStreamSynchronize(strm(c)));
  return GS_OK;
}

int gs_debug_attention(gs_ctx* c, const void* q, const void* k, const void* v, void* o, int heads, int d, int q_rs,
                       int kv_rs, int o_rs, const int* seq_off, const int* seq_len, int nreq) {
  if (!c || !seq_off || !seq_len) return GS_EINVAL;
  std::lock_guard<std::mutex> g(c->api_mu);
  RET(no_runs_in_flight(c, "gs_debug_attention"));
  CK(cudaSetDevice(c->device));
  RET(order_after_legacy(c));
  cudaError_t err = attention_tc(q, k, v, o, heads, d, q_rs, kv_rs, o_rs, seq_off, seq_len, nreq, c->num_sms, strm(c));
  if (err != cudaSuccess) return fail(c, err == cudaErrorInvalidValue ? GS_EINVAL : GS_ECUDA, "attention: %s", cudaGetErrorString(err));
  CK(cudaStreamSynchronize(strm(c)));
  return GS_OK;
}

int gs_debug_time_embed(gs_ctx* c, int model, int nreq, const float* t, float* e0, float* e) {
  if (!c || !t || !e0 || !e) return GS_EINVAL;
  std::lock_guard<std::mutex> g(c->api_mu);
  RET(no_runs_in_flight(c, "gs_debug_time_embed"));
  CK(cudaSetDevice(c->device));
  if (model < 0 || model >= static_cast<int>(c->models.size())) return fail(c, GS_EINVAL, "bad model id");
  if (nreq < 1 || nreq > MAX_BATCH) return fail(c, GS_EINVAL, "nreq");
  Model* m = c->models[model].get();
  RankArena& A = c->local[0];
  const int D = m->desc.dim;
  RET(ensure(c, A.e0, MAX_BATCH * D * 4));
  RET(ensure(c, A.e, MAX_BATCH * 6 * D * 4));
  RET(ensure(c, A.temb, (MAX_BATCH * m->desc.freq_dim + 2 * MAX_BATCH * D) * 4));
  TimeEmbedW tw{m->w_t1, m->b_t1, m->w_t2, m->b_t2, m->w_tp, m->b_tp, D, m->desc.freq_dim};
  CK(time_embed(tw, nreq, t, A.temb.as<float>(), A.e0.as<float>(), A.e.as<float>(), strm(c)));
  CK(cudaMemcpyAsync(e0, A.e0.p, static_cast<size_t>(nreq) * D * 4, cudaMemcpyDeviceToHost, strm(c)));
  CK(cudaMemcpyAsync(e, A.e.p, static_cast<size_t>(nreq) * 6 * D * 4, cudaMemcpyDeviceToHost, strm(c)));
  CK(cudaStreamSynchronize(strm(c)));
  return GS_OK;
}

int gs_debug_block(gs_ctx* c, int model, int layer, float* x, int nreq, const int* grids, const int* tok_lo,
                   const int* n_rows, const float* t, const void* prompts) {
  if (!c || !x || !grids || !tok_lo || !n_rows || !t) return GS_EINVAL;
  std::lock_guard<std::mutex> g(c->api_mu);
  RET(no_runs_in_flight(c, "gs_debug_block"));
  CK(cudaSetDevice(c->device));
  if (model < 0 || model >= static_cast<int>(c->models.size())) return fail(c, GS_EINVAL, "bad model id");
  Model* m = c->models[model].get();
  if (layer < 0 || layer >= m->desc.layers) return fail(c, GS_EINVAL, "bad layer");
  if (nreq < 1 || nreq > MAX_BATCH) return fail(c, GS_EINVAL, "nreq");
  // A p = 1 plan over segments [tok_lo, tok_lo + n_rows) of each request; attention runs over
  // the segment only (pass full requests, tok_lo = 0, for the block of the method).
  if (m->desc.cross_attn && !prompts) return fail(c, GS_EINVAL, "cross-attention model: prompts required");
  std::vector<std::unique_ptr<Request>> own(nreq);
  std::vector<Request*> reqs(nreq);
  const size_t psz = static_cast<size_t>(m->desc.text_len) * m->desc.text_dim;
  for (int r = 0; r < nreq; ++r) {
    own[r] = std::make_unique<Request>();
    for (int a = 0; a < 3; ++a) own[r]->grid[a] = grids[3 * r + a];
    own[r]->n = n_rows[r];
    own[r]->steps = 1;
    if (m->desc.cross_attn) {
      const uint16_t* pp = static_cast<const uint16_t*>(prompts) + r * psz;
      own[r]->prompt_host.assign(pp, pp + psz);
      RET(ensure_text_cache(c, m, own[r].get(), 0));
    }
    reqs[r] = own[r].get();
  }
  int rank0 = c->local[0].rank;
  Plan P;
  make_plan(P, m, reqs, &rank0, 1);
  RankArena& A = c->local[0];
  RET(prepare_rank(c, P, 0, A));
  // row_tok = tok_lo + local index
  {
    std::vector<int> rt(P.rows[0]);
    for (int r = 0; r < nreq; ++r)
      for (int i = 0; i < n_rows[r]; ++i) rt[P.loff[0][r] + i] = tok_lo[r] + i;
    CK(cudaMemcpyAsync(A.row_tok.p, rt.data(), rt.size() * 4, cudaMemcpyHostToDevice, strm(c)));
    CK(cudaStreamSynchronize(strm(c)));
  }
  const int D = m->desc.dim;
  TimeEmbedW tw{m->w_t1, m->b_t1, m->w_t2, m->b_t2, m->w_tp, m->b_tp, D, m->desc.freq_dim};
  CK(time_embed(tw, nreq, t, A.temb.as<float>(), A.e0.as<float>(), A.e.as<float>(), strm(c)));
  const size_t xbytes = static_cast<size_t>(P.rows[0]) * D * 4;
  CK(cudaMemcpyAsync(A.x.p, x, xbytes, cudaMemcpyHostToDevice, strm(c)));
  RET(block_pre(c, P, 0, A, layer));
  RET(block_attn(c, P, 0, A));
  RET(block_post(c, P, 0, A, layer));
  CK(cudaMemcpyAsync(x, A.x.p, xbytes, cudaMemcpyDeviceToHost, strm(c)));
  CK(cudaStreamSynchronize(strm(c)));
  for (auto& q : own) free_text_cache(c, q.get());
  prof_flush(c);
  return GS_OK;
}

}  // extern "C"
