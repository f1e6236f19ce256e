// Element-wise / row-wise kernels of the DiT step (HBM-bound; SURVEY.md §8(a) rows a2, a4, a6,
// a11, a14): LayerNorm + adaLN modulate, qk-RMSNorm + 3-axis RoPE + Ulysses send-layout pack,
// the time-embedding MLP (tiny GEMVs), fp32 -> bf16 conversion.
//
// Every row reduction uses a fixed order that depends only on D (thread-strided partial sums,
// xor-shuffle tree, then warp partials summed in warp order), so a row's result does not
// depend on where the row sits in the batch (SURVEY.md §8(a) invariant 2).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <map>
#include <mutex>
#include <tuple>
#include <cstdlib>

#include "kernels.h"
#include "ptx.cuh"

namespace gs {
namespace {

constexpr int ROW_THREADS = 128;
constexpr int MAXV = 16;  // float4 / uint4 per thread per row -> D <= 8192

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Sum over the NW warps of the CTA in a fixed order (pairwise tree in warp order); result
// broadcast to all threads.
template <int NW = 4>
__device__ __forceinline__ float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  if (NW == 4) return (red[0] + red[1]) + (red[2] + red[3]);
  return ((red[0] + red[1]) + (red[2] + red[3])) + ((red[4] + red[5]) + (red[6] + red[7]));
}

// Row kernels come in three shapes, chosen by D alone (so every row of a model takes the same
// reduction order): TPR = 256 threads per row (one row per CTA, D > 2048: Wan-14B), TPR = 64 (two
// warps per row, 8 rows per CTA, 1024 < D <= 2048: Wan-1.3B) or TPR = 32 (a warp per row, 8 rows
// per CTA, shuffle-only reductions, D <= 1024).  One CTA per row left HBM half idle at the
// config-2 T2I shape (26% of peak).
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
// TPR = 64 (two warps per row, 8 rows per CTA): warp sums exchanged through red[2 * slot + w]
// (warp order), one named barrier per row slot.  red holds >= 16 floats.
template <int TPR>
__device__ __forceinline__ float row_sum(float v, float* red) {
  if (TPR == 32) return warp_sum(v);
  if (TPR == 64) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, slot = w >> 1;
    named_bar_sync(1 + slot, 64);  // the partner has read the previous exchange
    if ((threadIdx.x & 31) == 0) red[2 * slot + (w & 1)] = v;
    named_bar_sync(1 + slot, 64);
    return red[2 * slot] + red[2 * slot + 1];
  }
  return block_sum<TPR / 32>(v, red);
}
// Two row sums at once (q and k of the qk kernel): the same per-value order as two row_sum calls
// (identical bits), one exchange instead of two -- the kernel is bound by these latency chains.
template <int TPR>
__device__ __forceinline__ float2 row_sum2(float a, float b, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if (TPR == 32) return make_float2(a, b);
  const int w = threadIdx.x >> 5;
  if (TPR == 64) {
    const int slot = w >> 1;
    named_bar_sync(1 + slot, 64);  // the partner has read the previous exchange
    if ((threadIdx.x & 31) == 0) {
      red[4 * slot + (w & 1)] = a;
      red[4 * slot + 2 + (w & 1)] = b;
    }
    named_bar_sync(1 + slot, 64);
    return make_float2(red[4 * slot] + red[4 * slot + 1], red[4 * slot + 2] + red[4 * slot + 3]);
  }
  constexpr int NW = TPR / 32;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
    red[w] = a;
    red[NW + w] = b;
  }
  __syncthreads();
  if (NW == 4)
    return make_float2((red[0] + red[1]) + (red[2] + red[3]), (red[4] + red[5]) + (red[6] + red[7]));
  return make_float2(((red[0] + red[1]) + (red[2] + red[3])) + ((red[4] + red[5]) + (red[6] + red[7])),
                     ((red[8] + red[9]) + (red[10] + red[11])) + ((red[12] + red[13]) + (red[14] + red[15])));
}
constexpr int kWarpRowMaxD = 2048;
constexpr int kWarpRowsPerCta = 8;

// ------------------------------------------------------------------ LN + modulate
// VPL = float4 (LN) / uint4 per tensor (qk) per thread: sized exactly from D so the registers of
// one row stay small and several CTAs share an SM (occupancy hides the DRAM latency of the row).
// Each row op is split into a load-and-sum half and a finish half (a persistent variant that
// streamed rows through shared memory by bulk copies reused them; it was slower, notes r01g).
template <int TPR, int VPL>
__device__ __forceinline__ float ln_load(const float4* xr, int tid, int nv, float4 (&v)[VPL]) {
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int c = tid + i * TPR;
    if (c < nv) {
      v[i] = xr[c];
      s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
    }
  }
  return s;
}

template <int TPR, int VPL, bool STAGED = false>
__device__ __forceinline__ void ln_finish(const float4 (&v)[VPL], float s, long long row, int tid, int D,
                                          const float* __restrict__ sh_a, const float* __restrict__ sh_b,
                                          const float* __restrict__ sc_a, const float* __restrict__ sc_b,
                                          int b_stride, const int* __restrict__ row_req, float eps,
                                          __nv_bfloat16* __restrict__ out, float* red,
                                          const float4* shs = nullptr, const float4* scs = nullptr) {
  const int nv = D >> 2;
  const float mean = row_sum<TPR>(s, red) / D;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int c = tid + i * TPR;
    if (c < nv) {
      const float a = v[i].x - mean, b = v[i].y - mean, cc = v[i].z - mean, d = v[i].w - mean;
      q += (a * a + b * b) + (cc * cc + d * d);
    }
  }
  const float rstd = rsqrtf(row_sum<TPR>(q, red) / D + eps);
  const int r = row_req[row];
  const float4* sha = reinterpret_cast<const float4*>(sh_a);
  const float4* sca = reinterpret_cast<const float4*>(sc_a);
  const float4* shb = reinterpret_cast<const float4*>(sh_b + (long long)r * b_stride);
  const float4* scb = reinterpret_cast<const float4*>(sc_b + (long long)r * b_stride);
  uint2* o = reinterpret_cast<uint2*>(out + row * D);
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int c = tid + i * TPR;
    if (c < nv) {
      float4 sh, sc;  // sh_a + sh_b[r], 1 + (sc_a + sc_b[r]): from the CTA's shared copy when staged
      if (STAGED) {
        sh = shs[c];
        sc = scs[c];
      } else {
        const float4 a1 = __ldg(sha + c), b1 = __ldg(shb + c), a2 = __ldg(sca + c), b2 = __ldg(scb + c);
        sh = make_float4(a1.x + b1.x, a1.y + b1.y, a1.z + b1.z, a1.w + b1.w);
        sc = make_float4(1.f + (a2.x + b2.x), 1.f + (a2.y + b2.y), 1.f + (a2.z + b2.z), 1.f + (a2.w + b2.w));
      }
      const float y0 = (v[i].x - mean) * rstd * sc.x + sh.x;
      const float y1 = (v[i].y - mean) * rstd * sc.y + sh.y;
      const float y2 = (v[i].z - mean) * rstd * sc.z + sh.z;
      const float y3 = (v[i].w - mean) * rstd * sc.w + sh.w;
      __nv_bfloat162 p0 = __floats2bfloat162_rn(y0, y1), p1 = __floats2bfloat162_rn(y2, y3);
      o[c] = make_uint2(*reinterpret_cast<uint32_t*>(&p0), *reinterpret_cast<uint32_t*>(&p1));
    }
  }
}

// Grid-stride over row groups (RPC rows per CTA per iteration).  When a group's rows belong to one request (rows
// are request segments, so all but the groups at a request boundary), the combined shift / 1 + scale vectors of
// that request are formed in shared memory (dynamic, 2 D floats) and kept while the CTA's next groups belong to
// the same request: per row 2 shared-memory float4 reads per 4 elements instead of 4 L1 loads and 8 adds (the same
// fp32 operations, hence the same bits).
template <int TPR, int VPL, int MINB>
__global__ void __launch_bounds__(TPR < 128 ? TPR * kWarpRowsPerCta : TPR, MINB)
    ln_modulate_kernel(const float* __restrict__ x, int M, int D, const float* __restrict__ sh_a,
                       const float* __restrict__ sh_b, const float* __restrict__ sc_a,
                       const float* __restrict__ sc_b, int b_stride, const int* __restrict__ row_req,
                       float eps, __nv_bfloat16* __restrict__ out) {
  __shared__ float red[16];
  extern __shared__ float4 ln_stage[];  // [D / 4] shift, then [D / 4] 1 + scale
  pdl_wait();
  pdl_launch_dependents();
  constexpr int RPC = TPR < 128 ? kWarpRowsPerCta : 1;
  const int nv = D >> 2;
  const int tid = TPR < 128 ? (threadIdx.x & (TPR - 1)) : threadIdx.x;
  float4* s_sh = ln_stage;
  float4* s_sc = ln_stage + nv;
  int staged_r = -1;  // request whose vectors the stage holds (CTA-uniform)
  for (long long row0 = static_cast<long long>(blockIdx.x) * RPC; row0 < M;
       row0 += static_cast<long long>(gridDim.x) * RPC) {
    const long long row = row0 + (TPR < 128 ? threadIdx.x / TPR : 0);
    const long long rlast = row0 + RPC - 1 < M ? row0 + RPC - 1 : M - 1;
    float4 v[VPL];
    float s = 0.f;
    if (row < M) s = ln_load<TPR, VPL>(reinterpret_cast<const float4*>(x + row * D), tid, nv, v);
    const int r0 = row_req[row0];
    const bool staged = r0 == row_req[rlast];
    if (staged && r0 != staged_r) {
      __syncthreads();  // every reader of the previous request's vectors is done
      const float4* sha = reinterpret_cast<const float4*>(sh_a);
      const float4* sca = reinterpret_cast<const float4*>(sc_a);
      const float4* shb = reinterpret_cast<const float4*>(sh_b + (long long)r0 * b_stride);
      const float4* scb = reinterpret_cast<const float4*>(sc_b + (long long)r0 * b_stride);
      for (int c = threadIdx.x; c < nv; c += blockDim.x) {
        const float4 a1 = __ldg(sha + c), b1 = __ldg(shb + c), a2 = __ldg(sca + c), b2 = __ldg(scb + c);
        s_sh[c] = make_float4(a1.x + b1.x, a1.y + b1.y, a1.z + b1.z, a1.w + b1.w);
        s_sc[c] = make_float4(1.f + (a2.x + b2.x), 1.f + (a2.y + b2.y), 1.f + (a2.z + b2.z), 1.f + (a2.w + b2.w));
      }
      __syncthreads();
      staged_r = r0;
    }
    if (TPR >= 128 || row < M) {
      if (staged)
        ln_finish<TPR, VPL, true>(v, s, row, tid, D, sh_a, sh_b, sc_a, sc_b, b_stride, row_req, eps, out, red, s_sh,
                                  s_sc);
      else
        ln_finish<TPR, VPL>(v, s, row, tid, D, sh_a, sh_b, sc_a, sc_b, b_stride, row_req, eps, out, red);
    }
  }
}

// ------------------------------------------------------------------ qk-RMSNorm + RoPE + pack
__device__ __forceinline__ void unpack8(const uint4& u, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}

// Per-CTA lookup tables of the pack / RoPE mapping, built once per CTA instead of searched per
// 8-element chunk (the qk kernel is instruction-bound: ncu issue-active 36% at 12% warps active):
// head h -> pack chunk jc, heads in the chunk hn, head index within the chunk hr; RoPE pair slot ->
// axis (0 = f, 1 = h, 2 = w).
constexpr int kMaxHeads = 128;  // D <= 8192, d >= 64
constexpr int kMaxSlots = 64;   // d / 2, d <= 128
struct QkTables {
  uint8_t jc[kMaxHeads], hn[kMaxHeads], hr[kMaxHeads], ax[kMaxSlots];
};

__device__ __forceinline__ void qk_tables_build(QkTables& t, const PackParams& pk, const RopeParams& rp, int H,
                                                int half) {
  for (int h = threadIdx.x; h < H; h += blockDim.x) {
    int jc = 0;
    for (int j = 1; j < pk.ndest; ++j)
      if (h >= pk.head_off[j]) jc = j;
    t.jc[h] = (uint8_t)jc;
    t.hn[h] = (uint8_t)(pk.head_off[jc + 1] - pk.head_off[jc]);
    t.hr[h] = (uint8_t)(h - pk.head_off[jc]);
  }
  for (int j = threadIdx.x; j < half; j += blockDim.x) t.ax[j] = (uint8_t)rp.slot_axis[j];
  __syncthreads();
}

// bf16 pair word -> (lo, hi) as fp32 (exact)
__device__ __forceinline__ float2 bf2f(uint32_t w) {
  return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
}
// Sum of squares of the 8 bf16 values of a chunk: ((f0^2 + f1^2) + (f2^2 + f3^2)) + ((f4^2 + f5^2) + (f6^2 + f7^2)),
// the even / odd halves of each word as the two lanes of packed FMUL2 / FFMA2.
__device__ __forceinline__ float sumsq8(const uint4& u) {
  const float2 a = bf2f(u.x), b = bf2f(u.y), c = bf2f(u.z), e = bf2f(u.w);
  const float2 ab = __ffma2_rn(make_float2(a.y, b.y), make_float2(a.y, b.y), __fmul2_rn(make_float2(a.x, b.x),
                                                                                         make_float2(a.x, b.x)));
  const float2 ce = __ffma2_rn(make_float2(c.y, e.y), make_float2(c.y, e.y), __fmul2_rn(make_float2(c.x, e.x),
                                                                                         make_float2(c.x, e.x)));
  return (ab.x + ab.y) + (ce.x + ce.y);
}
// One bf16 pair (x0, x1) of q or k: y = (x * r) * g (RMSNorm with gain), then the RoPE rotation
// (y0 c - y1 s, y0 s + y1 c) with ncs = (-s, c), cs = (c, s); packed to a bf16 pair word.
__device__ __forceinline__ uint32_t norm_rope_pair(uint32_t xw, uint32_t gw, float2 r2, float2 cs, float2 ncs) {
  const float2 y = __fmul2_rn(__fmul2_rn(bf2f(xw), r2), bf2f(gw));
  const float2 t = __fmul2_rn(make_float2(y.y, y.y), ncs);  // (-y1 s, y1 c)
  const float2 o = __ffma2_rn(make_float2(y.x, y.x), cs, t);
  return pack_bf16x2(o.x, o.y);
}

// One row per (TPR threads) per iteration; the CTA loops over rows (grid-stride) so the lookup tables and the
// per-thread constants (gain / RoPE slots, the same for every row: TPR * 8 is a multiple of d) are set up once
// per CTA instead of once per row.  v is copied to its destination unless v_out == nullptr in the plain
// (non-peer) layout: at SP = 1 the attention reads V in place from the QKV GEMM output.
template <int TPR, int VPL, int MINB>
__global__ void __launch_bounds__(TPR < 128 ? TPR * kWarpRowsPerCta : TPR, MINB)
    qk_norm_rope_pack_kernel(const __nv_bfloat16* __restrict__ qkv, int M, int D, int d,
                             const __nv_bfloat16* __restrict__ g_q, const __nv_bfloat16* __restrict__ g_k,
                             float eps, const RopeParams rp, const PackParams pk,
                             __nv_bfloat16* __restrict__ q_out, __nv_bfloat16* __restrict__ k_out,
                             __nv_bfloat16* __restrict__ v_out) {
  __shared__ float red[32];  // row_sum2: 4 per row slot (TPR = 64, 8 slots) or 2 x 8 warps
  __shared__ QkTables tb;
  pdl_wait();
  pdl_launch_dependents();
  const int half = d >> 1;
  qk_tables_build(tb, pk, rp, D / d, half);
  constexpr int RPC = TPR < 128 ? kWarpRowsPerCta : 1;  // rows per CTA per iteration
  const int tid = TPR < 128 ? (threadIdx.x & (TPR - 1)) : threadIdx.x;
  const int nv = D >> 3;
  const int lgd = __ffs(d) - 1;  // d in {64, 128}
  const int i0 = (tid * 8) & (d - 1);  // element offset within the head: the same for all chunks of this thread
  int ax[4];
#pragma unroll
  for (int p = 0; p < 4; ++p) ax[p] = tb.ax[(i0 >> 1) + p];
  const bool copy_v = pk.peer || v_out != nullptr;
  const uint4* gq = reinterpret_cast<const uint4*>(g_q);
  const uint4* gk = reinterpret_cast<const uint4*>(g_k);
  for (long long row = static_cast<long long>(blockIdx.x) * RPC + (TPR < 128 ? threadIdx.x / TPR : 0); row < M;
       row += static_cast<long long>(gridDim.x) * RPC) {
    const uint4* src = reinterpret_cast<const uint4*>(qkv + row * 3LL * D);
    uint4 qv[VPL], kv[VPL];
    float sq = 0.f, sk = 0.f;
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const int c = tid + i * TPR;
      if (c < nv) {
        qv[i] = src[c];
        kv[i] = src[nv + c];
        sq += sumsq8(qv[i]);
        sk += sumsq8(kv[i]);
      }
    }
    const int r = rp.row_req[row];
    const int tok = rp.row_tok[row];
    const int Ht = rp.req_grid[3 * r + 1], Wt = rp.req_grid[3 * r + 2];
    const int pos[3] = {tok / (Ht * Wt), (tok / Wt) % Ht, tok % Wt};
    float2 cs[4], ncs[4];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const int a = ax[p];
      cs[p] = __ldg(rp.cs_tab + static_cast<long long>(a == 0 ? pos[0] : (a == 1 ? pos[1] : pos[2])) * half +
                    (i0 >> 1) + p);
      ncs[p] = make_float2(-cs[p].y, cs[p].x);
    }
    long long prow = row;  // destination row
    if (pk.peer) {
      int sqi = 0;
      for (int t = 1; t < pk.nseq; ++t)
        if (row >= pk.seq_lo[t]) sqi = t;
      prow = row + pk.row_delta[sqi];
    }
    const float2 ssum = row_sum2<TPR>(sq, sk, red);
    const float rq = rsqrtf(ssum.x / D + eps);
    const float rk = rsqrtf(ssum.y / D + eps);
    const float2 rq2 = make_float2(rq, rq), rk2 = make_float2(rk, rk);
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const int c = tid + i * TPR;
      if (c < nv) {
        const int h = (c * 8) >> lgd;
        const int jc = tb.jc[h], hn = tb.hn[h], hr = tb.hr[h];
        __nv_bfloat16 *dq = q_out, *dk = k_out, *dv = v_out;
        long long o = (prow * hn + hr) * (long long)d + i0;
        if (pk.peer) {
          dq = pk.dst_q[jc];
          dk = pk.dst_k[jc];
          dv = pk.dst_v[jc];
        } else {
          o += pk.dest_off[jc];
        }
        const uint4 wq = __ldg(gq + c), wk = __ldg(gk + c);
        uint4 oq, ok;
        oq.x = norm_rope_pair(qv[i].x, wq.x, rq2, cs[0], ncs[0]);
        oq.y = norm_rope_pair(qv[i].y, wq.y, rq2, cs[1], ncs[1]);
        oq.z = norm_rope_pair(qv[i].z, wq.z, rq2, cs[2], ncs[2]);
        oq.w = norm_rope_pair(qv[i].w, wq.w, rq2, cs[3], ncs[3]);
        ok.x = norm_rope_pair(kv[i].x, wk.x, rk2, cs[0], ncs[0]);
        ok.y = norm_rope_pair(kv[i].y, wk.y, rk2, cs[1], ncs[1]);
        ok.z = norm_rope_pair(kv[i].z, wk.z, rk2, cs[2], ncs[2]);
        ok.w = norm_rope_pair(kv[i].w, wk.w, rk2, cs[3], ncs[3]);
        *reinterpret_cast<uint4*>(dq + o) = oq;
        *reinterpret_cast<uint4*>(dk + o) = ok;
        if (copy_v) *reinterpret_cast<uint4*>(dv + o) = src[2 * nv + c];
      }
    }
  }
}

// Streaming form for D > 1024 (kQkStreamMinD): a warp per row, grid-stride over rows, no block barrier.  Pass 1
// streams q and k from HBM (U chunks per lane in flight) and forms the lane's sums of squares (chunks in lane
// order, then the xor-shuffle tree: a fixed order that depends on D alone); pass 2 re-reads the row (L2-resident:
// the warp read it a moment ago) and writes the normalised, rotated q and k (and v, unless it stays in place).
// Few registers per row, so many rows are in flight per SM: the row-per-CTA form above is bound by its per-row
// latency chain (load -> block reduction -> compute -> store) at ~3 rows per SM.
// SSQ (D > 2048, qk_uses_ssq): the sums come from the QKV GEMM epilogue's per-32-column partials instead of pass 1,
// so q and k are read once.
constexpr int kQkStreamMinD = 1025;
#ifndef GS_QK_U
#define GS_QK_U 2  // pass-1 chunks per lane in flight
#endif
#ifndef GS_QK_SSQ_MINB
#define GS_QK_SSQ_MINB 4  // resident CTAs per SM of the single-pass form (64 registers)
#endif
constexpr int kQkStreamWarps = 8;  // warps (rows) per CTA
template <int U, bool SSQ>
__global__ void __launch_bounds__(32 * kQkStreamWarps, SSQ ? GS_QK_SSQ_MINB : 3)
    qk_norm_rope_stream_kernel(const __nv_bfloat16* __restrict__ qkv, int M, int D, int d,
                               const __nv_bfloat16* __restrict__ g_q, const __nv_bfloat16* __restrict__ g_k,
                               float eps, const RopeParams rp, const PackParams pk,
                               __nv_bfloat16* __restrict__ q_out, __nv_bfloat16* __restrict__ k_out,
                               __nv_bfloat16* __restrict__ v_out, const float* __restrict__ ssq) {
  __shared__ QkTables tb;
  pdl_wait();
  pdl_launch_dependents();
  const int half = d >> 1;
  qk_tables_build(tb, pk, rp, D / d, half);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nv = D >> 3;
  const int lgd = __ffs(d) - 1;
  const int i0 = (lane * 8) & (d - 1);  // the same for every chunk of this lane (256 is a multiple of d)
  int ax[4];
#pragma unroll
  for (int p = 0; p < 4; ++p) ax[p] = tb.ax[(i0 >> 1) + p];
  const bool copy_v = pk.peer || v_out != nullptr;
  const uint4* gq = reinterpret_cast<const uint4*>(g_q);
  const uint4* gk = reinterpret_cast<const uint4*>(g_k);
  // pass 1 marks the row's lines evict-last so they survive in L2 until pass 2 re-reads them (without the hint
  // ~75% of the pass-2 reads missed at config 4: DRAM reads 1.76x the algorithmic bytes, 2.73 GB -> 2.13 GB with
  // it); pass 2 releases them
  const uint64_t keep = l2_policy_evict_last(), drop = l2_policy_evict_first();
  for (long long row = static_cast<long long>(blockIdx.x) * kQkStreamWarps + warp; row < M;
       row += static_cast<long long>(gridDim.x) * kQkStreamWarps) {
    const uint4* src = reinterpret_cast<const uint4*>(qkv + row * 3LL * D);
    float sq = 0.f, sk = 0.f;
    if constexpr (SSQ) {
      // the QKV GEMM's per-32-column sums of squares (lane-strided, then the xor tree below): q and k are read once
      const int nc = D >> 5;
      const float* sr = ssq + row * 2LL * nc;
      for (int c = lane; c < nc; c += 32) {
        sq += sr[c];
        sk += sr[nc + c];
      }
    } else {
    // pass 1: sums of squares
    for (int c0 = lane; c0 < nv; c0 += 32 * U) {
      uint4 qv[U], kv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = c0 + 32 * u;
        if (c < nv) {
          qv[u] = ldg_l2hint(src + c, keep);
          kv[u] = ldg_l2hint(src + nv + c, keep);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (c0 + 32 * u < nv) {
          sq += sumsq8(qv[u]);
          sk += sumsq8(kv[u]);
        }
    }
    }
    // per-row constants (overlap the reduction)
    const int r = rp.row_req[row];
    const int tok = rp.row_tok[row];
    const int Ht = rp.req_grid[3 * r + 1], Wt = rp.req_grid[3 * r + 2];
    const int pos[3] = {tok / (Ht * Wt), (tok / Wt) % Ht, tok % Wt};
    float2 cs[4];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const int a = ax[p];
      cs[p] = __ldg(rp.cs_tab + static_cast<long long>(a == 0 ? pos[0] : (a == 1 ? pos[1] : pos[2])) * half +
                    (i0 >> 1) + p);
    }
    long long prow = row;
    if (pk.peer) {
      int sqi = 0;
      for (int t = 1; t < pk.nseq; ++t)
        if (row >= pk.seq_lo[t]) sqi = t;
      prow = row + pk.row_delta[sqi];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sq += __shfl_xor_sync(0xffffffffu, sq, o);
      sk += __shfl_xor_sync(0xffffffffu, sk, o);
    }
    const float rq = rsqrtf(sq / D + eps), rk = rsqrtf(sk / D + eps);
    const float2 rq2 = make_float2(rq, rq), rk2 = make_float2(rk, rk);
    // pass 2: normalise, rotate, store; the next chunk's q / k (and v) are loaded before this one is computed
    uint4 q = ldg_l2hint(src + lane, drop), k = ldg_l2hint(src + nv + lane, drop);
    uint4 v = copy_v ? ldg_l2hint(src + 2 * nv + lane, drop) : make_uint4(0, 0, 0, 0);
#pragma unroll 1
    for (int c = lane; c < nv; c += 32) {
      uint4 qn = q, kn = k, vn = v;
      if (c + 32 < nv) {
        qn = ldg_l2hint(src + c + 32, drop);
        kn = ldg_l2hint(src + nv + c + 32, drop);
        if (copy_v) vn = ldg_l2hint(src + 2 * nv + c + 32, drop);
      }
      const int h = (c * 8) >> lgd;
      const int jc = tb.jc[h], hn = tb.hn[h], hr = tb.hr[h];
      __nv_bfloat16 *dq = q_out, *dk = k_out, *dv = v_out;
      long long o = (prow * hn + hr) * (long long)d + i0;
      if (pk.peer) {
        dq = pk.dst_q[jc];
        dk = pk.dst_k[jc];
        dv = pk.dst_v[jc];
      } else {
        o += pk.dest_off[jc];
      }
      const uint4 wq = __ldg(gq + c), wk = __ldg(gk + c);
      uint4 oq, ok;
      oq.x = norm_rope_pair(q.x, wq.x, rq2, cs[0], make_float2(-cs[0].y, cs[0].x));
      oq.y = norm_rope_pair(q.y, wq.y, rq2, cs[1], make_float2(-cs[1].y, cs[1].x));
      oq.z = norm_rope_pair(q.z, wq.z, rq2, cs[2], make_float2(-cs[2].y, cs[2].x));
      oq.w = norm_rope_pair(q.w, wq.w, rq2, cs[3], make_float2(-cs[3].y, cs[3].x));
      ok.x = norm_rope_pair(k.x, wk.x, rk2, cs[0], make_float2(-cs[0].y, cs[0].x));
      ok.y = norm_rope_pair(k.y, wk.y, rk2, cs[1], make_float2(-cs[1].y, cs[1].x));
      ok.z = norm_rope_pair(k.z, wk.z, rk2, cs[2], make_float2(-cs[2].y, cs[2].x));
      ok.w = norm_rope_pair(k.w, wk.w, rk2, cs[3], make_float2(-cs[3].y, cs[3].x));
      *reinterpret_cast<uint4*>(dq + o) = oq;
      *reinterpret_cast<uint4*>(dk + o) = ok;
      if (copy_v) *reinterpret_cast<uint4*>(dv + o) = v;
      q = qn;
      k = kn;
      v = vn;
    }
  }
}

// ------------------------------------------------------------------ time embedding
struct TVals {
  float t[8];
};

__global__ void sinusoid_kernel(TVals tv, int B, int freq_dim, float* out) {
  const int half = freq_dim / 2;
  for (int i = threadIdx.x; i < B * half; i += blockDim.x) {
    const int b = i / half, j = i - b * half;
    const double w = exp(-log(10000.0) * (double)j / (double)half);
    const double a = (double)tv.t[b] * w;
    out[b * freq_dim + j] = (float)cos(a);
    out[b * freq_dim + half + j] = (float)sin(a);
  }
}

// y[b, n] = sum_k W[n, k] in[b, k] + bias[n]; one warp per output n, B <= 8.
__global__ void gemv_kernel(const float* __restrict__ in, const __nv_bfloat16* __restrict__ W,
                            const __nv_bfloat16* __restrict__ bias, int N, int K, int B,
                            float* __restrict__ out, float* __restrict__ out_silu) {
  const int n = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (n >= N) return;
  float acc[8];
#pragma unroll
  for (int b = 0; b < 8; ++b) acc[b] = 0.f;
  const __nv_bfloat162* w2 = reinterpret_cast<const __nv_bfloat162*>(W + (long long)n * K);
  for (int k2 = lane; k2 < K / 2; k2 += 32) {
    const float2 w = __bfloat1622float2(w2[k2]);
#pragma unroll
    for (int b = 0; b < 8; ++b)
      if (b < B) acc[b] += w.x * in[b * K + 2 * k2] + w.y * in[b * K + 2 * k2 + 1];
  }
  const float bn = __bfloat162float(bias[n]);
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    if (b < B) {
      const float y = warp_sum(acc[b]) + bn;
      if (lane == 0) {
        if (out) out[b * N + n] = y;
        if (out_silu) out_silu[b * N + n] = y / (1.f + __expf(-y));
      }
    }
  }
}

__global__ void f32_to_bf16_kernel(const float* __restrict__ in, __nv_bfloat16* __restrict__ out,
                                   long long n4) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    const float4 v = reinterpret_cast<const float4*>(in)[i];
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    reinterpret_cast<uint2*>(out)[i] =
        make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
  }
}

__global__ void __launch_bounds__(ROW_THREADS)
    rmsnorm_rows_kernel(const __nv_bfloat16* __restrict__ in, int ld_in, int D, const __nv_bfloat16* __restrict__ g,
                        float eps, __nv_bfloat16* __restrict__ out) {
  __shared__ float red[4];
  const long long row = blockIdx.x;
  const int nv = D >> 3;
  const uint4* src = reinterpret_cast<const uint4*>(in + row * ld_in);
  uint4 xv[MAXV / 2];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < MAXV / 2; ++i) {
    const int c = threadIdx.x + i * ROW_THREADS;
    if (c < nv) {
      xv[i] = src[c];
      float f[8];
      unpack8(xv[i], f);
      ss += ((f[0] * f[0] + f[1] * f[1]) + (f[2] * f[2] + f[3] * f[3])) +
            ((f[4] * f[4] + f[5] * f[5]) + (f[6] * f[6] + f[7] * f[7]));
    }
  }
  const float r = rsqrtf(block_sum(ss, red) / D + eps);
  const uint4* gv = reinterpret_cast<const uint4*>(g);
  uint4* dst = reinterpret_cast<uint4*>(out + row * D);
#pragma unroll
  for (int i = 0; i < MAXV / 2; ++i) {
    const int c = threadIdx.x + i * ROW_THREADS;
    if (c < nv) {
      float f[8], w[8];
      unpack8(xv[i], f);
      unpack8(__ldg(gv + c), w);
      dst[c] = make_uint4(pack_bf16x2(f[0] * r * w[0], f[1] * r * w[1]), pack_bf16x2(f[2] * r * w[2], f[3] * r * w[3]),
                          pack_bf16x2(f[4] * r * w[4], f[5] * r * w[5]), pack_bf16x2(f[6] * r * w[6], f[7] * r * w[7]));
    }
  }
}

__global__ void cfg_euler_kernel(float* __restrict__ z, float* __restrict__ z2, const float* __restrict__ vc,
                                 const float* __restrict__ vu, long long n, float dsig, float g) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const float v = vu ? vu[i] + g * (vc[i] - vu[i]) : vc[i];
    const float zn = z[i] + dsig * v;
    z[i] = zn;
    if (z2) z2[i] = zn;  // the uncond branch's copy of the shared latent
  }
}

}  // namespace

cudaError_t rmsnorm_rows(const __nv_bfloat16* in, int ld_in, int M, int D, const __nv_bfloat16* g, float eps,
                         __nv_bfloat16* out, cudaStream_t stream) {
  if (M == 0) return cudaSuccess;
  if (D % 8 || ld_in % 8 || D > 8 * (MAXV / 2) * ROW_THREADS) return cudaErrorInvalidValue;
  rmsnorm_rows_kernel<<<M, ROW_THREADS, 0, stream>>>(in, ld_in, D, g, eps, out);
  return cudaGetLastError();
}

cudaError_t cfg_euler(float* z, float* z2, const float* vc, const float* vu, long long n, float dsig, float g,
                      cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  cfg_euler_kernel<<<(int)blocks, 256, 0, stream>>>(z, z2, vc, vu, n, dsig, g);
  return cudaGetLastError();
}

std::atomic<int> g_pdl{-1};  // -1: not yet read from GS_PDL (default on)

bool pdl_enabled() {
  int v = g_pdl.load(std::memory_order_relaxed);
  if (v < 0) {
    v = (getenv("GS_PDL") && getenv("GS_PDL")[0] == '0') ? 0 : 1;
    g_pdl.store(v);
  }
  return v != 0;
}

namespace {
// Launch with the programmatic-dependent-launch attribute (when enabled).
template <class K, class... Args>
cudaError_t launch_pdl(K kernel, dim3 grid, dim3 block, cudaStream_t stream, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr.val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

template <class K, class... Args>
cudaError_t launch_pdl_smem(K kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t stream, Args... args) {
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) != cudaSuccess)
    return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr.val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

// Grid of a grid-stride row kernel: as many CTAs as are resident at once (per-CTA set-up done once), never more
// than there are row groups.
// (resident CTAs per device, cached per kernel / device / block / shared-memory size: the occupancy query is a
// host-side cost on every launch otherwise)
template <class K>
dim3 resident_grid(K kern, dim3 block, size_t smem, long long units) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, unsigned, size_t>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(reinterpret_cast<const void*>(kern), dev, block.x, smem);
  int resident = 0;
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) resident = it->second;
  }
  if (resident == 0) {
    int nb = 0, nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, block.x, smem) != cudaSuccess || nb < 1) nb = 1;
    resident = nb * std::max(nsm, 1);
    std::lock_guard<std::mutex> g(mu);
    cache[key] = resident;
  }
  return dim3(static_cast<unsigned>(std::min<long long>(units, resident)));
}

// Threads per row, from D alone (every row of a model takes the same reduction order).  Two warps
// per row for 1024 < D <= 2048 (Wan-1.3B): half the registers per thread, 32 instead of 24
// resident warps per SM; config 2 (r01k, same box) LN 2.72 -> 2.41, qk 2.54 -> 2.37 ms per step.
int row_tpr(int D) {
  // D > 2048 (Wan-14B): 256 threads per row (r01p: config 4 LN 41.3 -> 40.2, qk 58.6 -> 56.2 ms/step)
  if (D > kWarpRowMaxD) return 256;
  return D > 1024 ? 64 : 32;
}
}  // namespace

cudaError_t ln_modulate(const float* x, int M, int D, const float* sh_a, const float* sh_b,
                        const float* sc_a, const float* sc_b, int b_stride, const int* row_req,
                        float eps, __nv_bfloat16* out, cudaStream_t stream) {
  if (M == 0) return cudaSuccess;
  if (D % 4 || D > 4 * MAXV * ROW_THREADS) return cudaErrorInvalidValue;
  const int tpr = row_tpr(D);
  const int vpl = (D / 4 + tpr - 1) / tpr;  // 1..16
  const long long units = tpr < 128 ? (M + kWarpRowsPerCta - 1) / kWarpRowsPerCta : M;
  const dim3 block(tpr < 128 ? tpr * kWarpRowsPerCta : tpr);
  const size_t smem = 2ull * D * sizeof(float);  // the staged shift / 1 + scale vectors
#define GS_LN_CASE(T, V)                                                                                       \
  case V: {                                                                                                    \
    auto kern = ln_modulate_kernel<T, V, T == 32 ? 3 : (T == 64 ? 2 : (T == 256 ? 3 : 1))>;                  \
    if (cudaError_t e = launch_pdl_smem(kern, resident_grid(kern, block, smem, units), block, smem, stream, x, M, D, \
                                        sh_a, sh_b, sc_a, sc_b, b_stride, row_req, eps, out))                   \
      return e;                                                                                                 \
    break;                                                                                                      \
  }
#define GS_LN_SWITCH(T)                                                                                     \
  switch (vpl) {                                                                                           \
    GS_LN_CASE(T, 1) GS_LN_CASE(T, 2) GS_LN_CASE(T, 3) GS_LN_CASE(T, 4) GS_LN_CASE(T, 5) GS_LN_CASE(T, 6)  \
    GS_LN_CASE(T, 7) GS_LN_CASE(T, 8) GS_LN_CASE(T, 9) GS_LN_CASE(T, 10) GS_LN_CASE(T, 11)                 \
    GS_LN_CASE(T, 12) GS_LN_CASE(T, 13) GS_LN_CASE(T, 14) GS_LN_CASE(T, 15) GS_LN_CASE(T, 16)              \
    default: return cudaErrorInvalidValue;                                                                 \
  }
  if (tpr == 32) {
    GS_LN_SWITCH(32)
  } else if (tpr == 64) {
    switch (vpl) {
      GS_LN_CASE(64, 1) GS_LN_CASE(64, 2) GS_LN_CASE(64, 3) GS_LN_CASE(64, 4) GS_LN_CASE(64, 5)
      GS_LN_CASE(64, 6) GS_LN_CASE(64, 7) GS_LN_CASE(64, 8)
      default: return cudaErrorInvalidValue;
    }
  } else if (tpr == ROW_THREADS) {
    GS_LN_SWITCH(ROW_THREADS)
  } else if (tpr == 256) {
    switch (vpl) {
      GS_LN_CASE(256, 1) GS_LN_CASE(256, 2) GS_LN_CASE(256, 3) GS_LN_CASE(256, 4) GS_LN_CASE(256, 5)
      GS_LN_CASE(256, 6) GS_LN_CASE(256, 7) GS_LN_CASE(256, 8)
      default: return cudaErrorInvalidValue;
    }
  }
#undef GS_LN_SWITCH
#undef GS_LN_CASE
  return cudaGetLastError();
}

// Only above D = 2048: at config 2 (D = 1536, K = 1536) the extra epilogue work costs the QKV GEMM ~6 us per launch
// (164 -> 170 us), more than the 3.5 us the single-pass qk kernel saves (profiles/r02c/ssq/).
bool qk_uses_ssq(int D) { return D > kWarpRowMaxD; }

cudaError_t qk_norm_rope_pack(const __nv_bfloat16* qkv, int M, int D, int heads,
                              const __nv_bfloat16* g_q, const __nv_bfloat16* g_k, float eps,
                              const RopeParams& rp, const PackParams& pk, __nv_bfloat16* q_out,
                              __nv_bfloat16* k_out, __nv_bfloat16* v_out, cudaStream_t stream, const float* ssq) {
  if (M == 0) return cudaSuccess;
  const int d = D / heads;
  if (ssq != nullptr && (!qk_uses_ssq(D) || D % 32)) return cudaErrorInvalidValue;
  if (D % heads || d % 8 || D > 8 * (MAXV / 2) * ROW_THREADS || pk.ndest < 1 || pk.ndest > kMaxChunks)
    return cudaErrorInvalidValue;
  if (!pk.peer && (!q_out || !k_out)) return cudaErrorInvalidValue;
  if (D >= kQkStreamMinD) {
    auto kern = ssq ? qk_norm_rope_stream_kernel<GS_QK_U, true> : qk_norm_rope_stream_kernel<GS_QK_U, false>;
    const dim3 block(32 * kQkStreamWarps);
    return launch_pdl(kern, resident_grid(kern, block, 0, (M + kQkStreamWarps - 1) / kQkStreamWarps), block, stream,
                      qkv, M, D, d, g_q, g_k, eps, rp, pk, q_out, k_out, v_out, ssq);
  }
  const int tpr = row_tpr(D);
  const int vpl = (D / 8 + tpr - 1) / tpr;  // 1..8
  const long long units = tpr < 128 ? (M + kWarpRowsPerCta - 1) / kWarpRowsPerCta : M;
  const dim3 block(tpr < 128 ? tpr * kWarpRowsPerCta : tpr);
#define GS_QK_CASE(T, V)                                                                                     \
  case V: {                                                                                                  \
    auto kern = qk_norm_rope_pack_kernel<T, V, T == 32 ? 3 : (T == 64 ? 2 : (T == 256 ? 3 : 1))>;            \
    if (cudaError_t e = launch_pdl(kern, resident_grid(kern, block, 0, units), block, stream, qkv, M, D, d, g_q, g_k, eps, rp, pk,  \
                                   q_out, k_out, v_out))                                                     \
      return e;                                                                                               \
    break;                                                                                                   \
  }
#define GS_QK_SWITCH(T)                                                                                         \
  switch (vpl) {                                                                                               \
    GS_QK_CASE(T, 1) GS_QK_CASE(T, 2) GS_QK_CASE(T, 3) GS_QK_CASE(T, 4) GS_QK_CASE(T, 5) GS_QK_CASE(T, 6)      \
    GS_QK_CASE(T, 7) GS_QK_CASE(T, 8)                                                                          \
    default: return cudaErrorInvalidValue;                                                                     \
  }
  if (tpr == 32) {
    GS_QK_SWITCH(32)
  } else if (tpr == 64) {
    switch (vpl) {
      GS_QK_CASE(64, 1) GS_QK_CASE(64, 2) GS_QK_CASE(64, 3) GS_QK_CASE(64, 4)
      default: return cudaErrorInvalidValue;
    }
  } else if (tpr == ROW_THREADS) {
    GS_QK_SWITCH(ROW_THREADS)
  } else if (tpr == 256) {
    switch (vpl) {
      GS_QK_CASE(256, 1) GS_QK_CASE(256, 2) GS_QK_CASE(256, 3) GS_QK_CASE(256, 4)
      default: return cudaErrorInvalidValue;
    }
  }
#undef GS_QK_SWITCH
#undef GS_QK_CASE
  return cudaGetLastError();
}

// ------------------------------------------------------------------ peer barrier
__global__ void peer_signal_kernel(const PeerFlags f) {
  const int t = threadIdx.x;
  if (t < f.n) {
    // order every store this device made before (the producing kernels, earlier on the stream)
    // ahead of the flag at system scope, then publish the flag with release semantics
    asm volatile("fence.sc.sys;" ::: "memory");
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f.slot[t]), "l"(f.val[t]) : "memory");
  }
}

__global__ void peer_wait_kernel(const PeerFlags f) {
  const int t = threadIdx.x;
  if (t < f.n) {
    unsigned long long v = 0;
    const long long t0 = clock64();
    for (;;) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(f.slot[t]) : "memory");
      if (v >= f.val[t]) break;
      if (clock64() - t0 > 40000000000LL) __trap();  // ~20 s at 2 GHz: a peer died / mismatched plan
      __nanosleep(64);
    }
    asm volatile("fence.acq_rel.sys;" ::: "memory");
  }
  __syncthreads();
}

__global__ void peer_wait_probe_kernel(const PeerFlags f, long long timeout_ns, int* ok) {
  __shared__ int good;
  if (threadIdx.x == 0) good = 1;
  __syncthreads();
  const int t = threadIdx.x;
  if (t < f.n) {
    unsigned long long v = 0, t0, now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(f.slot[t]) : "memory");
      if (v >= f.val[t]) break;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (static_cast<long long>(now - t0) > timeout_ns) {
        atomicExch(&good, 0);
        break;
      }
      __nanosleep(256);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) *ok = good;
}

cudaError_t peer_wait_probe(const PeerFlags& f, int timeout_ms, int* ok, cudaStream_t stream) {
  if (f.n < 0 || f.n > 8 || !ok) return cudaErrorInvalidValue;
  peer_wait_probe_kernel<<<1, 32, 0, stream>>>(f, static_cast<long long>(timeout_ms) * 1000000LL, ok);
  return cudaGetLastError();
}

cudaError_t peer_signal(const PeerFlags& f, cudaStream_t stream) {
  if (f.n < 0 || f.n > 8) return cudaErrorInvalidValue;
  if (f.n == 0) return cudaSuccess;
  peer_signal_kernel<<<1, 32, 0, stream>>>(f);
  return cudaGetLastError();
}

cudaError_t peer_wait(const PeerFlags& f, cudaStream_t stream) {
  if (f.n < 0 || f.n > 8) return cudaErrorInvalidValue;
  if (f.n == 0) return cudaSuccess;
  peer_wait_kernel<<<1, 32, 0, stream>>>(f);
  return cudaGetLastError();
}

cudaError_t time_embed(const TimeEmbedW& w, int B, const float* t_host, float* scratch, float* e0,
                       float* e, cudaStream_t stream) {
  if (B < 1 || B > 8) return cudaErrorInvalidValue;
  TVals tv{};
  for (int b = 0; b < B; ++b) tv.t[b] = t_host[b];
  const int D = w.D, T = w.freq_dim;
  float* sin_buf = scratch;              // [B, T]
  float* h1 = scratch + 8 * T;           // [B, D]
  float* se0 = h1 + 8 * D;               // [B, D]
  sinusoid_kernel<<<1, 256, 0, stream>>>(tv, B, T, sin_buf);
  const int wpb = 8;  // warps per block
  gemv_kernel<<<(D + wpb - 1) / wpb, 32 * wpb, 0, stream>>>(sin_buf, w.w_t1, w.b_t1, D, T, B, nullptr, h1);
  gemv_kernel<<<(D + wpb - 1) / wpb, 32 * wpb, 0, stream>>>(h1, w.w_t2, w.b_t2, D, D, B, e0, se0);
  gemv_kernel<<<(6 * D + wpb - 1) / wpb, 32 * wpb, 0, stream>>>(se0, w.w_tp, w.b_tp, 6 * D, D, B, e, nullptr);
  return cudaGetLastError();
}

cudaError_t f32_to_bf16(const float* in, __nv_bfloat16* out, long long n, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  if (n % 4) return cudaErrorInvalidValue;
  long long blocks = (n / 4 + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  f32_to_bf16_kernel<<<(int)blocks, 256, 0, stream>>>(in, out, n / 4);
  return cudaGetLastError();
}

}  // namespace gs
