// tcgen05 flash attention, non-causal, varlen block-diagonal:
//   O_h = softmax(Q_h K_h^T / sqrt(d)) V_h per request (oracle: oracle/dit.py attention()).
//
// Design (B200-first; FlashAttention-4-style structure, written from scratch):
//   * one CTA = one head x two 128-row Q tiles of one request (256 query rows); for d = 128 two
//     CTAs form a pair (cta_group::2, M = 256 MMAs issued by the leader, see Cfg);
//   * warps 0..3 / 4..7: softmax warpgroups WG0 / WG1, one thread per query row;
//   * warp 8: TMA producer (Q once; K_j and V_j into rings of Cfg::KST / Cfg::VST slots, 128B
//     swizzle);
//   * warp 9: TMEM owner + single-thread tcgen05.mma issuer (warps 10, 11 idle);
//   * griddepcontrol.wait after the setup (programmatic dependent launch, ptx.cuh);
//   * TMEM (512 cols): S_w = Q_w K_j^T at cols [128w, 128w+128) (fp32), P_w (bf16 pairs)
//     written over S_w cols [128w, 128w+64), O_w at cols [256+128w, 256+128w+d);
//   * MMA issue order S0_0, S1_0, {PV0_j, S0_{j+1}, PV1_j, S1_{j+1}}: WG0's softmax of tile j+1
//     overlaps PV1_j / S1_{j+1} on the tensor core and vice versa (ping-pong);
//   * online softmax in fp32 (exp2 domain) with lazy rescale: O is rescaled only when the
//     running max grows by more than 2^8 (values stay <= 256 otherwise, exact in fp32).
// Bit-exactness (SURVEY.md §8(a) invariant 3): Q and KV tiles start at each request's first
// token, the KV loop always covers the request in the same order, tiles never mix requests
// (out-of-request columns are masked to p = 0).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "kernels.h"
#include "ptx.cuh"
#include "tma.h"

namespace gs {
// Development trace (GS_ATTN_TRACE=1): clock64 stamps of CTA (0,0) for the first 32 KV tiles.
__device__ unsigned long long g_attn_trace[2 * 16 * 64];  // [CTA 0 / its pair peer][event][tile][group]
// Development trace (GS_ATTN_TRACE=1): per CTA (linear id < 8192) globaltimer at entry / after the
// prologue (first S issued) / exit, and the SM id -- per-CTA overhead and inter-CTA gaps.
__device__ unsigned long long g_attn_ctatime[8192 * 4];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
namespace {
#define TRACE_EV(ev, w, j) \
  if (TRACE && blockIdx.x < 2 && blockIdx.y == 0 && (j) < 32) \
    g_attn_trace[blockIdx.x * 1024 + ((ev) * 32 + (j)) * 2 + (w)] = clock64()

constexpr int MAX_REQ = 64;
constexpr int THREADS = 384;
// Warp roles.  The SMSP arbiter issues highest-warp-id first, so the latency-critical producer
// and MMA-issuer warps take the highest ids (8, 9) and are never starved by the softmax warps
// (0-3: Q tile 0, 4-7: Q tile 1) sharing their SMSPs; warps 10, 11 idle.
constexpr int kProducerWarp = 8, kMmaWarp = 9;

struct SeqTable {
  int nreq;
  int q_off[MAX_REQ], q_len[MAX_REQ];    // query rows of segment r
  int kv_off[MAX_REQ], kv_len[MAX_REQ];  // key / value rows it attends to (= q for self-attention)
  int tile_start[MAX_REQ + 1];           // prefix sum of ceil(q_len / rows per CTA (pair))
};

// PAIR (d = 128): CTA pairs with cta_group::2 MMAs (M = 256 = both CTAs' Q tile w): each CTA stages
// half of every K tile (64 keys, the B operand's N half) and half of every V tile (64 of the d
// columns), halving per-SM shared-memory B reads and L2 -> SM traffic (tools/micro: the UMMA smem
// read path is 128 B/clk).
template <int HD, bool PAIR>
struct Cfg {
  static constexpr int BOXES = HD / 64;                  // 64-element (128 B) column boxes
  static constexpr int TILE_BYTES = 128 * HD * 2;        // one 128-row Q tile
  static constexpr int KT_BYTES = (PAIR ? 64 : 128) * HD * 2;       // this CTA's part of a K tile
  static constexpr int KBOX_BYTES = (PAIR ? 64 : 128) * 128;       // one [rows][64] K box
  static constexpr int VT_BYTES = 128 * (PAIR ? HD / 2 : HD) * 2;  // this CTA's part of a V tile
  // K ring deeper than V: a K slot frees after both S MMAs, a V slot only after both PV MMAs
  static constexpr int KST = PAIR ? 4 : (HD == 128 ? 3 : 4);
  static constexpr int VST = PAIR ? 4 : (HD == 128 ? 2 : 4);
  static constexpr int Q_OFF = 0;
  static constexpr int K_OFF = 2 * TILE_BYTES;
  static constexpr int V_OFF = K_OFF + KST * KT_BYTES;
  static constexpr int BAR_OFF = V_OFF + VST * VT_BYTES;
  static constexpr int SMEM = BAR_OFF + 256 + 1024;
};


// Which of every 8 exp2 pairs go to the FMA-pipe polynomial: spread out so the polynomial's FMA /
// ALU instructions fill the 8-cycle MUFU issue gaps of the neighbouring pairs.
template <int POLY8>
__device__ __forceinline__ constexpr bool poly_pair(int k) {
  return POLY8 == 0 ? false
       : POLY8 == 2 ? (k == 2 || k == 6)
       : POLY8 == 3 ? (k == 1 || k == 4 || k == 6)
       : (k & 1) == 1;
}

// P = exp2(S * scale - m) for the 128 columns of this thread's row, packed to bf16 pairs and
// stored over the S columns [0, 64) in TMEM (P aliases S).  Returns the fp32 partial row sums.
// FULL = false is the last (partial) KV tile of a request: masked columns get p = 0 exactly.
// KEEP: also write the fp32 p values back over v (the row sum is then taken after the P hand-off,
// off the softmax -> MMA chain; -DGS_ATTN_LSUM=1) and return zeros.
template <int POLY8, bool FULL, int NCOL = 128, bool KEEP = false>
__device__ __forceinline__ float2 exp_pack_store(uint32_t (&v)[NCOL], float2 sc2, float2 nm2,
                                                 int kv_valid, uint32_t tS, int col0 = 0) {
  float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
#pragma unroll
  for (int c = 0; c < NCOL / 32; ++c) {
    uint32_t pk[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int col = c * 32 + 2 * i;
      const float2 x =
          __ffma2_rn(make_float2(__uint_as_float(v[col]), __uint_as_float(v[col + 1])), sc2, nm2);
      // exp2: MUFU for most pairs, FMA-pipe polynomial for POLY8 of every 8 pairs (reading 22)
      float2 p;
      if (poly_pair<POLY8>(i & 7)) {
        p = exp2_poly2(x);
      } else {
        p.x = ex2_approx(x.x);
        p.y = ex2_approx(x.y);
      }
      if (!FULL) {
        p.x = col0 + col < kv_valid ? p.x : 0.f;
        p.y = col0 + col + 1 < kv_valid ? p.y : 0.f;
      }
      if (KEEP) {
        v[col] = __float_as_uint(p.x);
        v[col + 1] = __float_as_uint(p.y);
      } else if (i & 1) {
        acc1 = __fadd2_rn(acc1, p);
      } else {
        acc0 = __fadd2_rn(acc0, p);
      }
      pk[i] = pack_bf16x2(p.x, p.y);
    }
    GS_TMEM_ST16(tS + c * 16, pk);
  }
  return __fadd2_rn(acc0, acc1);
}

// SCATTER: the fused head->seq exchange epilogue (OScatter); a separate instantiation so the plain
// kernel keeps its register allocation (the scatter lookup in the shared epilogue cost ~5%).
// SPLITP (-DGS_ATTN_SPLITP=1, development A/B): the softmax hands P over in two 64-key halves so the
// issuer can start PV on the first half while the second is still being exponentiated.
#ifndef GS_ATTN_SPLITP
#define GS_ATTN_SPLITP 0
#endif
constexpr int NPH = GS_ATTN_SPLITP ? 2 : 1;  // P hand-offs per group per KV tile
// SEQ (-DGS_ATTN_SEQ=1, development A/B): phase lock between the two softmax warpgroups through two
// named barriers -- WG1 pauses after the first 64 keys of its exps until WG0 has handed over its
// whole P of the same tile, and WG0 continues past its hand-off only once WG1 reached that midpoint,
// so WG1 runs half a softmax behind WG0 and the two never drift into lock-step.
#ifndef GS_ATTN_SEQ
#define GS_ATTN_SEQ 0
#endif
// LSUM (-DGS_ATTN_LSUM=1, development A/B): the row sum of p is taken after P is handed over.
#ifndef GS_ATTN_LSUM
#define GS_ATTN_LSUM 0
#endif
constexpr bool kSeq = GS_ATTN_SEQ != 0, kLsum = GS_ATTN_LSUM != 0;
constexpr int kBarSeqA = 1, kBarSeqB = 2;  // named barrier ids (0 = __syncthreads)

template <int HD, int POLY8, bool TRACE = false, bool PAIR = (HD == 128), bool SCATTER = false>
__global__ void __launch_bounds__(THREADS, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, __nv_bfloat16* __restrict__ O, int o_rs,
                   const __grid_constant__ SeqTable tab, float scale_log2,
                   const __grid_constant__ OScatter osc) {
  using C = Cfg<HD, PAIR>;
  const unsigned cta_lin = blockIdx.y * gridDim.x + blockIdx.x;
  if (TRACE && threadIdx.x == 0 && cta_lin < 8192) {
    g_attn_ctatime[cta_lin * 4 + 0] = gtimer();
    g_attn_ctatime[cta_lin * 4 + 3] = smid();
  }
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* q_full = bars;
  uint64_t* kfull = bars + 1;           // [KST]
  uint64_t* kempty = kfull + C::KST;    // [KST]
  uint64_t* vfull = kempty + C::KST;    // [VST]
  uint64_t* vempty = vfull + C::VST;    // [VST]
  uint64_t* sfull = vempty + C::VST;    // [2]
  uint64_t* pfull = sfull + 2;        // [2] (SPLITP: [2 groups][2 key halves])
  uint64_t* ofull = pfull + 2 * NPH;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ofull + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int head = blockIdx.y;
  const uint32_t rank = PAIR ? cluster_ctarank() : 0;  // 0 = leader (issues the MMAs)
  constexpr int ROWS = PAIR ? 512 : 256;               // query rows per CTA pair / CTA

  // locate (request, block of ROWS query rows) of this CTA (pair)
  const int blk = PAIR ? (blockIdx.x >> 1) : blockIdx.x;
  int r = 0;
  while (r + 1 < tab.nreq && blk >= tab.tile_start[r + 1]) ++r;
  const int pair = blk - tab.tile_start[r];
  const int kv_off = tab.kv_off[r], kv_len = tab.kv_len[r];
  const int q_row0 = tab.q_off[r] + pair * ROWS + rank * 256;
  const int q_rows = min(256, tab.q_len[r] - pair * ROWS - static_cast<int>(rank) * 256);  // may be <= 0
  const int nkv = (kv_len + 127) / 128;

  __shared__ int scat_meta[2];
  if (SCATTER && threadIdx.x == 0) {
    scat_meta[0] = r;
    scat_meta[1] = q_row0 - tab.q_off[r];
  }
  if (threadIdx.x == 0) {
    constexpr int NC = PAIR ? 2 : 1;  // leader-side full barriers count one arrival per CTA
    mbar_init(q_full, NC);
    for (int s = 0; s < C::KST; ++s) {
      mbar_init(&kfull[s], NC);
      mbar_init(&kempty[s], 1);
    }
    for (int s = 0; s < C::VST; ++s) {
      mbar_init(&vfull[s], NC);
      mbar_init(&vempty[s], 1);
    }
    for (int w = 0; w < 2; ++w) {
      mbar_init(&sfull[w], 1);
      for (int hh = 0; hh < NPH; ++hh) mbar_init(&pfull[w * NPH + hh], 4 * NC);
      mbar_init(&ofull[w], 1);
    }
    fence_barrier_init();
  }
  if (warp == kProducerWarp && lane == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
  }
  if (warp == kMmaWarp) {
    if (PAIR)
      tmem_alloc_2sm(tmem_slot, 512);
    else
      tmem_alloc(tmem_slot, 512);
  }
  tc_fence_before();
  if (PAIR)
    cluster_sync();  // both CTAs' barriers initialised before any remote arrive / 2-SM TMA
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // the setup above overlaps the previous kernel's tail; global memory only from here
  pdl_launch_dependents();

  // register split: producer / MMA warpgroup shrinks, the two softmax warpgroups grow.  The CTA
  // pool is 384 x 168 (launch allocation): 4 warps x 32 x (168 - 80) = 11264 freed >= 8 warps x
  // 32 x (208 - 168) = 10240 requested (an unsatisfiable .inc would block forever).
  if (warp >= 8) {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 80;");
  if (warp == kProducerWarp) {
    if (lane == 0) {
      // bytes land in this CTA's smem; the (leader's) full barrier counts them
      auto arrive_tx = [&](uint64_t* bar, uint32_t bytes) {
        if (PAIR)
          mbar_arrive_expect_tx_cluster(mapa_shared(smem_u32(bar), 0), bytes);
        else
          mbar_arrive_expect_tx(bar, bytes);
      };
      auto load = [&](const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1, int c2) {
        if (PAIR)
          tma_load_3d_2sm(map, bar, dst, c0, c1, c2);
        else
          tma_load_3d(map, bar, dst, c0, c1, c2);
      };
      arrive_tx(q_full, 2 * C::TILE_BYTES);
      for (int w = 0; w < 2; ++w)
        for (int b = 0; b < C::BOXES; ++b)
          load(&tmQ, q_full, smem + C::Q_OFF + w * C::TILE_BYTES + b * 16384, b * 64, head, q_row0 + w * 128);
      for (int j = 0; j < nkv; ++j) {
        const int ks = j % C::KST, vs = j % C::VST;
        mbar_wait(&kempty[ks], ((j / C::KST) & 1) ^ 1);
        uint8_t* sk = smem + C::K_OFF + ks * C::KT_BYTES;
        TRACE_EV(8, 0, j);
        arrive_tx(&kfull[ks], C::KT_BYTES);
        for (int b = 0; b < C::BOXES; ++b)  // PAIR: keys [64 rank, 64 rank + 64) of the tile
          load(&tmK, &kfull[ks], sk + b * C::KBOX_BYTES, b * 64, head, kv_off + j * 128 + (PAIR ? 64 * rank : 0));
        mbar_wait(&vempty[vs], ((j / C::VST) & 1) ^ 1);
        uint8_t* sv = smem + C::V_OFF + vs * C::VT_BYTES;
        TRACE_EV(9, 0, j);
        arrive_tx(&vfull[vs], C::VT_BYTES);
        if (PAIR)  // d columns [64 rank, 64 rank + 64) of all 128 keys
          load(&tmV, &vfull[vs], sv, 64 * rank, head, kv_off + j * 128);
        else
          for (int b = 0; b < C::BOXES; ++b)
            load(&tmV, &vfull[vs], sv + b * 16384, b * 64, head, kv_off + j * 128);
      }
    }
  } else if (warp == kMmaWarp && rank == 0) {
    // Single MMA issuer (the leader CTA of a pair).  Its fixed order PV0_j, S0_j+1, PV1_j, S1_j+1 keeps the two softmax
    // warpgroups half a period apart (ping-pong: one group's exp work overlaps the other's MMAs);
    // independent per-group issuers were measured to fall into lock-step (profiles/r01_notes.md).
    if (lane == 0) {
      constexpr uint32_t idesc_s = idesc_bf16(PAIR ? 256 : 128, 128, 0, 0);
      constexpr uint32_t idesc_o = idesc_bf16(PAIR ? 256 : 128, HD, 0, 1);
      auto commit = [&](uint64_t* bar) {
        if (PAIR)
          mma_commit_2sm_mc(bar, 0x3);
        else
          mma_commit(bar);
      };
      auto wait = [&](uint64_t* bar, uint32_t parity) { mbar_wait_spin(bar, parity); };
      const uint32_t sq = smem_u32(smem + C::Q_OFF);
      const uint32_t sk0 = smem_u32(smem + C::K_OFF);
      const uint32_t sv0 = smem_u32(smem + C::V_OFF);
      mbar_wait(q_full, 0);
      // issue without waiting: callers wait for K_j (kfull) / V_j (vfull) + P (pfull) first
      // descriptors: start-address field (addr >> 4, 14 bits) advanced by plain adds; smem < 256 KB so no carry
      const uint64_t qdesc0 = sdesc_sw128(sq, 16, 1024);
      const uint64_t kdesc0 = sdesc_sw128(sk0, 16, 1024);
      const uint64_t vdesc0 = sdesc_sw128(sv0, 16384, 1024);
      auto issue_s = [&](int w, int j) {  // S_w = Q_w K_j^T -> TMEM cols [128 w, 128 w + 128)
        TRACE_EV(0, w, j);
        const uint64_t qa = qdesc0 + ((w * C::TILE_BYTES) >> 4);
        const uint64_t kb = kdesc0 + (((j % C::KST) * C::KT_BYTES) >> 4);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t qoff = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
          const uint32_t koff = ((kk >> 2) * C::KBOX_BYTES + (kk & 3) * 32) >> 4;
          if (PAIR)
            mma_ss_2sm(tmem + w * 128, qa + qoff, kb + koff, idesc_s, kk > 0);
          else
            mma_ss(tmem + w * 128, qa + qoff, kb + koff, idesc_s, kk > 0);
        }
        commit(&sfull[w]);
        TRACE_EV(13, w, j);
      };
      auto issue_pv = [&](int w, int j, int half = -1) {  // O_w += P_w V_j, P_w from TMEM (bf16 over S_w)
        TRACE_EV(1, w, j);
        const uint64_t vb = vdesc0 + (((j % C::VST) * C::VT_BYTES) >> 4);
        const int k0 = half < 0 ? 0 : 4 * half, k1 = half < 0 ? 8 : k0 + 4;
#pragma unroll
        for (int kk = k0; kk < k1; ++kk) {
          if (PAIR)
            mma_ts_2sm(tmem + 256 + w * 128, tmem + w * 128 + kk * 8, vb + ((kk * 2048) >> 4), idesc_o,
                       (j > 0) || (kk > 0));
          else
            mma_ts(tmem + 256 + w * 128, tmem + w * 128 + kk * 8, vb + ((kk * 2048) >> 4), idesc_o,
                   (j > 0) || (kk > 0));
        }
        TRACE_EV(14, w, j);
      };
      auto wait_p = [&](int w, int j, int half = 0) {
        TRACE_EV(12, w, j);
        wait(&pfull[w * NPH + half], j & 1);
        TRACE_EV(10, w, j);
        tc_fence_after();
      };
      auto pv = [&](int w, int j) {  // wait for P_w and issue PV_w (in two halves with SPLITP)
        if (NPH == 2) {
          wait_p(w, j, 0);
          issue_pv(w, j, 0);
          wait_p(w, j, 1);
          issue_pv(w, j, 1);
        } else {
          wait_p(w, j);
          issue_pv(w, j);
        }
      };
      wait(&kfull[0], 0);
      tc_fence_after();
      if (TRACE && cta_lin < 8192) g_attn_ctatime[cta_lin * 4 + 1] = gtimer();
      issue_s(0, 0);
      issue_s(1, 0);
      commit(&kempty[0]);
      for (int j = 0; j < nkv; ++j) {
        const bool more = j + 1 < nkv;
        // V_j and K_{j+1} landed long ago in steady state: check them before waiting on P (folding
        // these checks into P0's barrier via a helper warp was measured: no gain, see r01_notes.md)
        TRACE_EV(15, 0, j);
        wait(&vfull[j % C::VST], (j / C::VST) & 1);
        if (more) wait(&kfull[(j + 1) % C::KST], ((j + 1) / C::KST) & 1);
        TRACE_EV(11, 0, j);
        pv(0, j);
        if (more) issue_s(0, j + 1);
        pv(1, j);
        commit(&vempty[j % C::VST]);
        if (more) {
          issue_s(1, j + 1);
          commit(&kempty[(j + 1) % C::KST]);
        }
      }
      commit(&ofull[0]);
      commit(&ofull[1]);
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;");
    const int w = warp >> 2;  // softmax warpgroup
    const int quarter = warp & 3;
    const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
    const uint32_t tS = tmem + lane_base + w * 128;
    const uint32_t tO = tmem + lane_base + 256 + w * 128;
    const float2 sc2 = make_float2(scale_log2, scale_log2);
    float m_run = -INFINITY, l_run = 0.f;
    for (int j = 0; j < nkv; ++j) {
      mbar_wait(&sfull[w], j & 1);
      tc_fence_after();
      if (quarter == 0 && lane == 0) TRACE_EV(2, w, j);
      const int kv_valid = min(128, kv_len - j * 128);
      // whole S row of this thread (128 fp32) in registers: one TMEM round trip per tile
      uint32_t v[128];
      GS_TMEM_LD32(tS + 0, (*reinterpret_cast<uint32_t(*)[32]>(v + 0)));
      GS_TMEM_LD32(tS + 32, (*reinterpret_cast<uint32_t(*)[32]>(v + 32)));
      GS_TMEM_LD32(tS + 64, (*reinterpret_cast<uint32_t(*)[32]>(v + 64)));
      GS_TMEM_LD32(tS + 96, (*reinterpret_cast<uint32_t(*)[32]>(v + 96)));
      tmem_ld_wait();
      if (quarter == 0 && lane == 0) TRACE_EV(3, w, j);
      const bool full = kv_valid == 128;  // warp-uniform: only a request's last tile is partial
      if (!full) {
#pragma unroll
        for (int i = 0; i < 128; ++i)
          if (i >= kv_valid) v[i] = __float_as_uint(-INFINITY);
      }
      // row max: 8 independent FMNMX3 chains (a 3-level tree over 128 values)
      float mx[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) mx[c] = fmax3(__uint_as_float(v[16 * c]), __uint_as_float(v[16 * c + 1]),
                                                __uint_as_float(v[16 * c + 2]));
#pragma unroll
      for (int i = 3; i < 15; i += 2)
#pragma unroll
        for (int c = 0; c < 8; ++c)
          mx[c] = fmax3(mx[c], __uint_as_float(v[16 * c + i]), __uint_as_float(v[16 * c + i + 1]));
#pragma unroll
      for (int c = 0; c < 8; ++c) mx[c] = fmaxf(mx[c], __uint_as_float(v[16 * c + 15]));
      const float m_tile =
          fmax3(fmax3(mx[0], mx[1], mx[2]), fmax3(mx[3], mx[4], mx[5]), fmaxf(mx[6], mx[7])) * scale_log2;
      // lazy rescale: move the reference max only when it grows by more than 2^8
      const bool need = m_tile > m_run + 8.0f;
      const float alpha = need ? ex2_approx(m_run - m_tile) : 1.0f;
      if (need) m_run = m_tile;
      if (j > 0 && __any_sync(0xffffffffu, need)) {
#pragma unroll 1
        for (int c = 0; c < HD / 32; ++c) {
          uint32_t o[32];
          GS_TMEM_LD32(tO + c * 32, o);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          GS_TMEM_ST32(tO + c * 32, o);
        }
      }
      l_run *= alpha;
      float2 acc;
      auto hand_over = [&](int hh) {  // P (or its half hh) is in TMEM: tell the MMA issuer
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (PAIR)
            mbar_arrive_cluster(mapa_shared(smem_u32(&pfull[w * NPH + hh]), 0));
          else
            mbar_arrive(&pfull[w * NPH + hh]);
        }
      };
      if (NPH == 2 || kSeq) {  // keys [0, 64) then [64, 128)
        uint32_t(&va)[64] = *reinterpret_cast<uint32_t(*)[64]>(v);
        uint32_t(&vb)[64] = *reinterpret_cast<uint32_t(*)[64]>(v + 64);
        const float2 nm2 = make_float2(-m_run, -m_run);
        float2 a0, a1;
        a0 = full ? exp_pack_store<POLY8, true, 64, kLsum>(va, sc2, nm2, kv_valid, tS, 0)
                  : exp_pack_store<POLY8, false, 64, kLsum>(va, sc2, nm2, kv_valid, tS, 0);
        if (NPH == 2) hand_over(0);  // the first half goes to the MMA issuer as soon as it is stored
        if (kSeq && w == 1) {        // WG1's midpoint: wait for WG0's hand-off of this tile
          asm volatile("bar.sync %0, 256;" ::"n"(kBarSeqB) : "memory");
          asm volatile("bar.arrive %0, 256;" ::"n"(kBarSeqA) : "memory");
        }
        a1 = full ? exp_pack_store<POLY8, true, 64, kLsum>(vb, sc2, nm2, kv_valid, tS + 32, 64)
                  : exp_pack_store<POLY8, false, 64, kLsum>(vb, sc2, nm2, kv_valid, tS + 32, 64);
        acc = __fadd2_rn(a0, a1);
      } else if (full) {
        acc = exp_pack_store<POLY8, true, 128, kLsum>(v, sc2, make_float2(-m_run, -m_run), kv_valid, tS);
      } else {
        acc = exp_pack_store<POLY8, false, 128, kLsum>(v, sc2, make_float2(-m_run, -m_run), kv_valid, tS);
      }
      if (!kLsum) l_run += acc.x + acc.y;
      const long long t_done = TRACE ? clock64() : 0;
      hand_over(NPH - 1);
      if (kSeq && w == 0) {  // WG0 past its hand-off: release WG1's midpoint, wait until WG1 is there
        asm volatile("bar.arrive %0, 256;" ::"n"(kBarSeqB) : "memory");
        asm volatile("bar.sync %0, 256;" ::"n"(kBarSeqA) : "memory");
      }
      if (kLsum) {  // row sum of this tile's p (fp32, kept in v), two chains
        float2 s0 = make_float2(0.f, 0.f), s1 = make_float2(0.f, 0.f);
#pragma unroll
        for (int i = 0; i < 64; i += 2) {
          s0 = __fadd2_rn(s0, make_float2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1])));
          s1 = __fadd2_rn(s1, make_float2(__uint_as_float(v[2 * i + 2]), __uint_as_float(v[2 * i + 3])));
        }
        acc = __fadd2_rn(s0, s1);
        l_run += acc.x + acc.y;
      }
      if (TRACE && lane == 0 && blockIdx.x < 2 && blockIdx.y == 0 && j < 32)
        g_attn_trace[blockIdx.x * 1024 + ((4 + quarter) * 32 + j) * 2 + w] = t_done;
    }
    // epilogue: O / l -> bf16 -> global
    mbar_wait(&ofull[w], 0);
    tc_fence_after();
    const int row_in = w * 128 + quarter * 32 + lane;
    const float inv = 1.0f / l_run;
    __nv_bfloat16* orow;
    if (SCATTER) {  // fused head->seq exchange: straight into the token owner's O-proj input
      // segment and first token of this CTA come back from shared memory (kept out of the
      // registers of the softmax loop)
      const int rr = scat_meta[0];
      const int t = scat_meta[1] + row_in;
      int i = 0;
#pragma unroll
      for (int k = 1; k < 8; ++k)
        if (k < osc.nown && t >= osc.lo[rr][k]) i = k;
      orow = osc.base[rr][i] + static_cast<long long>(t) * o_rs + head * HD;
    } else {
      orow = O + static_cast<long long>(q_row0 + row_in) * o_rs + head * HD;
    }
#pragma unroll
    for (int c = 0; c < HD / 32; ++c) {
      uint32_t v[32];
      GS_TMEM_LD32(tO + c * 32, v);
      tmem_ld_wait();
      if (row_in < q_rows) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i)
          pk[i] = pack_bf16x2(__uint_as_float(v[2 * i]) * inv, __uint_as_float(v[2 * i + 1]) * inv);
        uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
        for (int q = 0; q < 4; ++q) dst[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (PAIR) cluster_sync();  // the peer may still arrive on our barriers / read our TMEM until here
  if (warp == kMmaWarp) {
    __syncwarp();
    tc_fence_after();
    if (PAIR)
      tmem_dealloc_2sm(tmem, 512);
    else
      tmem_dealloc(tmem, 512);
  }
  if (TRACE && threadIdx.x == 0 && cta_lin < 8192) g_attn_ctatime[cta_lin * 4 + 2] = gtimer();
}

#ifndef GS_ATTN_ALT
#define GS_ATTN_ALT 0
#endif
#if GS_ATTN_ALT
// ---------------------------------------------------------------------------------------------
// v7 (d = 128, CTA pairs): one 128-row Q tile per CTA (M = 256 cta_group::2 MMAs per pair), KV
// tiles dealt alternately to two softmax warp sets (tile j -> set j & 1: warps 0-3 / 4-7, one
// thread per query row, the whole 128-column S row in registers), S / P in three TMEM buffers:
//   cols [0,128) O  |  [128 + 128 u, 256 + 128 u) S/P buffer u = j % 3  (P_j: bf16 pairs over
//   the buffer's first 64 columns, as in v5).
// The v5 chain (a Q tile's S_{j+1} waits for its own PV_j, which waits for its softmax) is gone:
// S_{j+2} only follows PV_{j-1}, the OTHER set's tile, so each set's softmax of tile j+2 can start
// as soon as its tile j is done, and the two sets keep the exp (MUFU) pipe and the tensor core
// busy at once.  The sets share one O accumulator, so they share the running max: set j & 1
// takes m_{j-1} from the other set (shared memory, one named barrier per warp pair), decides the
// lazy rescale of tile j (O rescaled only when the max grows by more than 2^8, after PV_{j-1}
// completed) and hands m_j on.  Each set keeps its partial row sum relative to the last max it
// saw; the epilogue brings both to the final max with the same exp2 factors O received.
//   warps 0-7: softmax, warp 8: TMA producer, warp 9: TMEM owner + MMA issuer (leader CTA), warps
//   10, 11 idle (setmaxnreg acts on whole warpgroups).
// Development variant (built with -DGS_ATTN_ALT=1; 12% slower than v5 at the c4 SP=8 shape in round 2).
constexpr int THREADS7 = 384;
constexpr int kProducerWarp7 = 8, kMmaWarp7 = 9, kSIssueWarp7 = 10;
struct Cfg7 {
  static constexpr int HD = 128;
  static constexpr int TILE_BYTES = 128 * HD * 2;   // this CTA's Q tile
  static constexpr int KT_BYTES = 64 * HD * 2;      // 64 of the tile's 128 keys
  static constexpr int KBOX_BYTES = 64 * 128;       // one [64 keys][64 d] box
  static constexpr int VT_BYTES = 128 * 64 * 2;     // 64 of the d columns of all 128 keys
  static constexpr int KST = 5, VST = 5;
  static constexpr int Q_OFF = 0;
  static constexpr int K_OFF = TILE_BYTES;
  static constexpr int V_OFF = K_OFF + KST * KT_BYTES;
  static constexpr int BAR_OFF = V_OFF + VST * VT_BYTES;
  static constexpr int XCH_OFF = BAR_OFF + 512;              // float [2 sets][128 rows] running max
  static constexpr int FIN_OFF = XCH_OFF + 2 * 128 * 4;      // float [2 sets][2 (l, m)][128 rows]
  static constexpr int SMEM = FIN_OFF + 2 * 2 * 128 * 4 + 1024;
  static constexpr uint32_t T_O = 0, T_S = 128;
};
static_assert(Cfg7::SMEM <= 232448, "v7 shared memory");

template <int POLY8, bool SCATTER, bool TRACE = false>
__global__ void __launch_bounds__(THREADS7, 1)
    attn_alt_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, __nv_bfloat16* __restrict__ O, int o_rs,
                    const __grid_constant__ SeqTable tab, float scale_log2, const __grid_constant__ OScatter osc) {
  using C = Cfg7;
  constexpr int HD = C::HD;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* q_full = bars;
  uint64_t* kfull = bars + 1;           // [KST]
  uint64_t* kempty = kfull + C::KST;    // [KST]
  uint64_t* vfull = kempty + C::KST;    // [VST]
  uint64_t* vempty = vfull + C::VST;    // [VST]
  uint64_t* sfull = vempty + C::VST;    // [3] S_j in buffer j % 3
  uint64_t* pfull = sfull + 3;          // [3] P_j in buffer j % 3 (leader: 8 warp arrivals)
  uint64_t* pvdone = pfull + 3;         // [3] PV_j completed
  uint64_t* pvis = pvdone + 3;          // [3] PV_j issued (PV issuer -> S issuer, leader CTA)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pvis + 3);
  float* xch = reinterpret_cast<float*>(smem + C::XCH_OFF);
  float* fin = reinterpret_cast<float*>(smem + C::FIN_OFF);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int head = blockIdx.y;
  const uint32_t rank = cluster_ctarank();  // 0 = leader (issues the MMAs)

  const int blk = blockIdx.x >> 1;
  int r = 0;
  while (r + 1 < tab.nreq && blk >= tab.tile_start[r + 1]) ++r;
  const int pair = blk - tab.tile_start[r];
  const int kv_off = tab.kv_off[r], kv_len = tab.kv_len[r];
  const int q_first = pair * 256 + static_cast<int>(rank) * 128;  // request-local first query row
  const int q_row0 = tab.q_off[r] + q_first;
  const int q_rows = min(128, tab.q_len[r] - q_first);  // may be <= 0
  const int nkv = (kv_len + 127) / 128;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 2);
    for (int s = 0; s < C::KST; ++s) {
      mbar_init(&kfull[s], 2);
      mbar_init(&kempty[s], 1);
    }
    for (int s = 0; s < C::VST; ++s) {
      mbar_init(&vfull[s], 2);
      mbar_init(&vempty[s], 1);
    }
    for (int u = 0; u < 3; ++u) {
      mbar_init(&sfull[u], 1);
      mbar_init(&pfull[u], 8);
      mbar_init(&pvdone[u], 1);
      mbar_init(&pvis[u], 1);
    }
    fence_barrier_init();
  }
  if (warp == kProducerWarp7 && lane == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
  }
  if (warp == kMmaWarp7) tmem_alloc_2sm(tmem_slot, 512);
  tc_fence_before();
  cluster_sync();  // both CTAs' barriers initialised before any remote arrive / 2-SM TMA
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // the setup above overlaps the previous kernel's tail; global memory only from here
  pdl_launch_dependents();

  // register split: the CTA pool is 384 x 168 (launch allocation); warpgroup 2 (producer, MMA, two
  // idle warps) shrinks to 56, freeing 4 x 32 x 112 = 14336 >= 8 x 32 x (208 - 168) = 10240.
  if (warp >= 8) {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
  if (warp == kProducerWarp7) {
    if (lane == 0) {
      auto arrive_tx = [&](uint64_t* bar, uint32_t bytes) {
        mbar_arrive_expect_tx_cluster(mapa_shared(smem_u32(bar), 0), bytes);
      };
      arrive_tx(q_full, C::TILE_BYTES);
      for (int b = 0; b < 2; ++b)
        tma_load_3d_2sm(&tmQ, q_full, smem + C::Q_OFF + b * 16384, b * 64, head, q_row0);
      for (int j = 0; j < nkv; ++j) {
        const int ks = j % C::KST, vs = j % C::VST;
        mbar_wait(&kempty[ks], ((j / C::KST) & 1) ^ 1);
        uint8_t* sk = smem + C::K_OFF + ks * C::KT_BYTES;
        arrive_tx(&kfull[ks], C::KT_BYTES);
        for (int b = 0; b < 2; ++b)  // keys [64 rank, 64 rank + 64) of the tile
          tma_load_3d_2sm(&tmK, &kfull[ks], sk + b * C::KBOX_BYTES, b * 64, head, kv_off + j * 128 + 64 * rank);
        mbar_wait(&vempty[vs], ((j / C::VST) & 1) ^ 1);
        arrive_tx(&vfull[vs], C::VT_BYTES);  // d columns [64 rank, 64 rank + 64) of all 128 keys
        tma_load_3d_2sm(&tmV, &vfull[vs], smem + C::V_OFF + vs * C::VT_BYTES, 64 * rank, head, kv_off + j * 128);
      }
    }
  } else if ((warp == kMmaWarp7 || warp == kSIssueWarp7) && rank == 0 && lane == 0) {
    // Two issuers in the leader CTA, on different SMSPs: warp 9 issues the PV MMAs, warp 10 the S MMAs,
    // so neither's barrier polls (~200 cycles each under MUFU load) leave the tensor core idle.  S_{j+3}
    // overwrites the buffer PV_j reads: the S issuer waits for "PV_j issued" (pvis, with the tcgen05
    // thread-sync fences), after which the in-order tensor core runs PV_j before S_{j+3}.
    constexpr uint32_t idesc_s = idesc_bf16(256, 128, 0, 0);
    constexpr uint32_t idesc_o = idesc_bf16(256, HD, 0, 1);
    const uint64_t qdesc0 = sdesc_sw128(smem_u32(smem + C::Q_OFF), 16, 1024);
    const uint64_t kdesc0 = sdesc_sw128(smem_u32(smem + C::K_OFF), 16, 1024);
    const uint64_t vdesc0 = sdesc_sw128(smem_u32(smem + C::V_OFF), 16384, 1024);
    if (warp == kSIssueWarp7) {
      auto issue_s = [&](int j) {  // S_j = Q K_j^T -> buffer j % 3; K slot and S_j signalled
        mbar_wait_spin(&kfull[j % C::KST], (j / C::KST) & 1);
        tc_fence_after();
        TRACE_EV(0, 0, j);
        const uint64_t kb = kdesc0 + (((j % C::KST) * C::KT_BYTES) >> 4);
        const uint32_t d = tmem + C::T_S + (j % 3) * 128;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t qoff = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
          const uint32_t koff = ((kk >> 2) * C::KBOX_BYTES + (kk & 3) * 32) >> 4;
          mma_ss_2sm(d, qdesc0 + qoff, kb + koff, idesc_s, kk > 0);
        }
        mma_commit_2sm_mc(&kempty[j % C::KST], 0x3);
        mma_commit_2sm_mc(&sfull[j % 3], 0x3);
      };
      mbar_wait(q_full, 0);
      for (int j = 0; j < 3 && j < nkv; ++j) issue_s(j);
      for (int j = 0; j + 3 < nkv; ++j) {
        mbar_wait_spin(&pvis[j % 3], (j / 3) & 1);  // PV_j is in the tensor core's queue
        tc_fence_after();
        issue_s(j + 3);
      }
    } else {
      for (int j = 0; j < nkv; ++j) {
        const int u = j % 3;
        mbar_wait_spin(&vfull[j % C::VST], (j / C::VST) & 1);
        TRACE_EV(7, 0, j);
        mbar_wait_spin(&pfull[u], (j / 3) & 1);
        tc_fence_after();
        TRACE_EV(1, 0, j);
        // O += P_j V_j, P_j read from TMEM (bf16 pairs over buffer u's first 64 columns)
        const uint64_t vb = vdesc0 + (((j % C::VST) * C::VT_BYTES) >> 4);
        const uint32_t pa = tmem + C::T_S + u * 128;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_ts_2sm(tmem + C::T_O, pa + kk * 8, vb + ((kk * 2048) >> 4), idesc_o, (j > 0) || (kk > 0));
        mma_commit_2sm_mc(&pvdone[u], 0x3);
        mma_commit_2sm_mc(&vempty[j % C::VST], 0x3);
        tc_fence_before();
        mbar_arrive(&pvis[u]);
      }
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;");
    const int set = warp >> 2, quarter = warp & 3;
    const int row_in = quarter * 32 + lane;
    const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
    const uint32_t tO = tmem + lane_base + C::T_O;
    const float2 sc2 = make_float2(scale_log2, scale_log2);
    const uint32_t pfull_leader = mapa_shared(smem_u32(&pfull[0]), 0);
    // named barriers 1-4: set 0 -> set 1 hand-off of the running max (per lane quarter); 5-8: set 1 -> set 0;
    // 9-12: the epilogue exchange of both sets' row sums
    const int bar_put = 1 + quarter + 4 * set, bar_get = 1 + quarter + 4 * (set ^ 1);
    float m_ref = -INFINITY, l_run = 0.f;  // this set's row sum, relative to exp2 max m_ref
    for (int j = set; j < nkv; j += 2) {
      const int u = j % 3;
      const uint32_t tS = tmem + lane_base + C::T_S + u * 128;
      mbar_wait(&sfull[u], (j / 3) & 1);
      tc_fence_after();
      if (quarter == 0 && lane == 0) TRACE_EV(2, 0, j);
      __syncwarp();
      const int kv_valid = min(128, kv_len - j * 128);
      uint32_t v[128];
      GS_TMEM_LD32(tS + 0, (*reinterpret_cast<uint32_t(*)[32]>(v + 0)));
      GS_TMEM_LD32(tS + 32, (*reinterpret_cast<uint32_t(*)[32]>(v + 32)));
      GS_TMEM_LD32(tS + 64, (*reinterpret_cast<uint32_t(*)[32]>(v + 64)));
      GS_TMEM_LD32(tS + 96, (*reinterpret_cast<uint32_t(*)[32]>(v + 96)));
      tmem_ld_wait();
      if (quarter == 0 && lane == 0) TRACE_EV(3, 0, j);
      const bool full = kv_valid == 128;  // warp-uniform: only a request's last tile is partial
      if (!full) {
#pragma unroll
        for (int i = 0; i < 128; ++i)
          if (i >= kv_valid) v[i] = __float_as_uint(-INFINITY);
      }
      float mx[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) mx[c] = fmax3(__uint_as_float(v[16 * c]), __uint_as_float(v[16 * c + 1]),
                                                __uint_as_float(v[16 * c + 2]));
#pragma unroll
      for (int i = 3; i < 15; i += 2)
#pragma unroll
        for (int c = 0; c < 8; ++c)
          mx[c] = fmax3(mx[c], __uint_as_float(v[16 * c + i]), __uint_as_float(v[16 * c + i + 1]));
#pragma unroll
      for (int c = 0; c < 8; ++c) mx[c] = fmaxf(mx[c], __uint_as_float(v[16 * c + 15]));
      const float m_tile =
          fmax3(fmax3(mx[0], mx[1], mx[2]), fmax3(mx[3], mx[4], mx[5]), fmaxf(mx[6], mx[7])) * scale_log2;
      // running max after tile j - 1 (the other set's tile)
      float m_prev = -INFINITY;
      if (quarter == 0 && lane == 0) TRACE_EV(4, 0, j);
      if (j > 0) {
        asm volatile("bar.sync %0, 64;" ::"r"(bar_get) : "memory");
        m_prev = xch[(set ^ 1) * 128 + row_in];
        if (m_prev != m_ref) {  // the other set moved the max at tile j - 1: same factor as O got
          l_run *= ex2_approx(m_ref - m_prev);
          m_ref = m_prev;
        }
      }
      // lazy rescale: move the reference max only when it grows by more than 2^8
      const bool need = m_tile > m_prev + 8.0f;
      const float alpha = need ? ex2_approx(m_prev - m_tile) : 1.0f;
      const float m_run = need ? m_tile : m_prev;
      if (j + 1 < nkv) {
        xch[set * 128 + row_in] = m_run;
        asm volatile("bar.arrive %0, 64;" ::"r"(bar_put) : "memory");
      }
      l_run *= alpha;
      m_ref = m_run;
      if (quarter == 0 && lane == 0) TRACE_EV(5, 0, j);
      __syncwarp();
      float2 acc;
      if (full)
        acc = exp_pack_store<POLY8, true>(v, sc2, make_float2(-m_run, -m_run), kv_valid, tS);
      else
        acc = exp_pack_store<POLY8, false>(v, sc2, make_float2(-m_run, -m_run), kv_valid, tS);
      l_run += acc.x + acc.y;
      if (quarter == 0 && lane == 0) TRACE_EV(6, 0, j);
      if (j > 0 && __any_sync(0xffffffffu, need)) {  // O holds PV_0..PV_{j-1}: rescale before PV_j
        mbar_wait(&pvdone[(j - 1) % 3], ((j - 1) / 3) & 1);
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < HD / 32; ++c) {
          uint32_t o[32];
          GS_TMEM_LD32(tO + c * 32, o);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          GS_TMEM_ST32(tO + c * 32, o);
        }
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(pfull_leader + u * 8);
      if (lane == 0) TRACE_EV(8 + quarter, 0, j);
      __syncwarp();
    }
    // row sum: both sets' partial sums brought to the final max m_ref of the set that did the last tile
    // The set of the last tile waits for the last PV before the exchange: its wait for S_{nkv-1}
    // implied PV_{nkv-4} (same buffer) done, so the parity test cannot alias an older phase; the
    // other set learns of the completion through the named barrier.
    const int last = (nkv - 1) & 1;
    fin[(set * 2 + 0) * 128 + row_in] = l_run;
    fin[(set * 2 + 1) * 128 + row_in] = m_ref;
    if (set == last) mbar_wait(&pvdone[(nkv - 1) % 3], ((nkv - 1) / 3) & 1);
    asm volatile("bar.sync %0, 64;" ::"r"(9 + quarter) : "memory");
    tc_fence_after();
    const float m_fin = fin[(last * 2 + 1) * 128 + row_in];
    float l_tot = 0.f;
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const float ls = fin[(s * 2 + 0) * 128 + row_in], ms = fin[(s * 2 + 1) * 128 + row_in];
      l_tot += ms == m_fin ? ls : ls * ex2_approx(ms - m_fin);
    }
    // epilogue: set s writes d columns [64 s, 64 s + 64)
    const float inv = 1.0f / l_tot;
    __nv_bfloat16* orow;
    if (SCATTER) {  // fused head->seq exchange: straight into the token owner's O-proj input
      const int t = q_first + row_in;
      int i = 0;
#pragma unroll
      for (int k = 1; k < 8; ++k)
        if (k < osc.nown && t >= osc.lo[r][k]) i = k;
      orow = osc.base[r][i] + static_cast<long long>(t) * o_rs + head * HD;
    } else {
      orow = O + static_cast<long long>(q_row0 + row_in) * o_rs + head * HD;
    }
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int col = set * 64 + c * 32;
      uint32_t v[32];
      GS_TMEM_LD32(tO + col, v);
      tmem_ld_wait();
      if (row_in < q_rows) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i)
          pk[i] = pack_bf16x2(__uint_as_float(v[2 * i]) * inv, __uint_as_float(v[2 * i + 1]) * inv);
        uint4* dst = reinterpret_cast<uint4*>(orow + col);
#pragma unroll
        for (int q = 0; q < 4; ++q) dst[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  cluster_sync();  // the peer may still arrive on our barriers / read our TMEM until here
  if (warp == kMmaWarp7) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc_2sm(tmem, 512);
  }
}

template <int POLY8>
cudaError_t launch_alt(const void* Q, const void* K, const void* V, void* O, int heads, int q_rs, int kv_rs,
                       int o_rs, const SeqTable& tab, int q_rows, int kv_rows, cudaStream_t stream,
                       const OScatter& osc) {
  using C = Cfg7;
  CUtensorMap tq, tk, tv;
  if (!make_tma_3d_bf16(&tq, Q, 128, heads, q_rows, 256ull, q_rs * 2ull, 64, 1, 128) ||
      !make_tma_3d_bf16(&tk, K, 128, heads, kv_rows, 256ull, kv_rs * 2ull, 64, 1, 64) ||
      !make_tma_3d_bf16(&tv, V, 128, heads, kv_rows, 256ull, kv_rs * 2ull, 64, 1, 128))
    return cudaErrorInvalidValue;
  static const bool trace = getenv("GS_ATTN_TRACE") != nullptr;
  auto kern = osc.nown > 0 ? attn_alt_kernel<POLY8, true>
              : trace      ? attn_alt_kernel<POLY8, false, true>
                           : attn_alt_kernel<POLY8, false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  if (e != cudaSuccess) return e;
  const float scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(128.0));
  dim3 grid(tab.tile_start[tab.nreq] * 2, heads);
  if (grid.x == 0) return cudaSuccess;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(THREADS7);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kern, tq, tk, tv, static_cast<__nv_bfloat16*>(O), o_rs, tab, scale_log2, osc);
}

#endif  // GS_ATTN_ALT
template <int HD, int POLY8>
cudaError_t launch_t(const void* Q, const void* K, const void* V, void* O, int heads, int q_rs,
                   int kv_rs, int o_rs, const SeqTable& tab, int q_rows, int kv_rows, cudaStream_t stream,
                   const OScatter& osc, int v_rs) {
  constexpr bool PAIR = HD == 128;
#if GS_ATTN_ALT
  if (HD == 128 && v_rs != kv_rs) return cudaErrorInvalidValue;
  if (HD == 128) return launch_alt<POLY8>(Q, K, V, O, heads, q_rs, kv_rs, o_rs, tab, q_rows, kv_rows, stream, osc);
#endif
  using C = Cfg<HD, PAIR>;
  CUtensorMap tq, tk, tv;
  if (!make_tma_3d_bf16(&tq, Q, HD, heads, q_rows, HD * 2ull, q_rs * 2ull, 64, 1, 128) ||
      !make_tma_3d_bf16(&tk, K, HD, heads, kv_rows, HD * 2ull, kv_rs * 2ull, 64, 1, PAIR ? 64 : 128) ||
      !make_tma_3d_bf16(&tv, V, HD, heads, kv_rows, HD * 2ull, v_rs * 2ull, 64, 1, 128))
    return cudaErrorInvalidValue;
  static const bool trace = getenv("GS_ATTN_TRACE") != nullptr;
  auto kern = osc.nown > 0 ? attn_tc_kernel<HD, POLY8, false, PAIR, true>
              : trace      ? attn_tc_kernel<HD, POLY8, true>
                           : attn_tc_kernel<HD, POLY8, false>;
  const int smem_bytes = C::SMEM;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
  if (e != cudaSuccess) return e;
  const float scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(HD)));
  dim3 grid(tab.tile_start[tab.nreq] * (PAIR ? 2 : 1), heads);
  if (grid.x == 0) return cudaSuccess;  // no query rows (an empty shard)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = smem_bytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = PAIR ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kern, tq, tk, tv, static_cast<__nv_bfloat16*>(O), o_rs, tab, scale_log2, osc);
}

// Fraction of exp2 pairs (in eighths) computed by the FMA-pipe polynomial: a compile-time constant
// (it changes output bits, so it must not differ between the processes of an SP group; the round-1
// sweep in profiles/r01_notes.md found 0 fastest).  Other values build with -DGS_ATTN_POLY8=2|3|4.
#ifndef GS_ATTN_POLY8
#define GS_ATTN_POLY8 0
#endif
static_assert(GS_ATTN_POLY8 == 0 || GS_ATTN_POLY8 == 2 || GS_ATTN_POLY8 == 3 || GS_ATTN_POLY8 == 4, "POLY8");

template <int HD>
cudaError_t launch(const void* Q, const void* K, const void* V, void* O, int heads, int q_rs,
                   int kv_rs, int o_rs, const SeqTable& tab, int q_rows, int kv_rows, cudaStream_t stream,
                   const OScatter& osc, int v_rs) {
  return launch_t<HD, GS_ATTN_POLY8>(Q, K, V, O, heads, q_rs, kv_rs, o_rs, tab, q_rows, kv_rows, stream, osc, v_rs);
}
}  // namespace

cudaError_t attention_tc_segments(const void* Q, const void* K, const void* V, void* O, int heads, int d,
                                  int q_rs, int kv_rs, int o_rs, const int* q_off, const int* q_len,
                                  const int* kv_off, const int* kv_len, int nreq, cudaStream_t stream,
                                  const OScatter* scatter, int v_rs) {
  if (v_rs == 0) v_rs = kv_rs;  // V's row stride (the QKV GEMM output's 3 D when V is read in place at SP = 1)
  if (nreq < 1 || nreq > MAX_REQ || (d != 64 && d != 128) || heads < 1) return cudaErrorInvalidValue;
  OScatter osc{};
  if (scatter && scatter->nown > 0) {
    if (nreq > OSC_MAX_REQ || scatter->nown > 8) return cudaErrorInvalidValue;
    osc = *scatter;
  }
  SeqTable tab{};
  tab.nreq = nreq;
  int q_rows = 1, kv_rows = 1;
  tab.tile_start[0] = 0;
  // a CTA pair (d = 128: two 128-row Q tiles per CTA) or a CTA (d = 64)
  const int rows_per_block = d == 128 ? (GS_ATTN_ALT ? 256 : 512) : 256;
  for (int r = 0; r < nreq; ++r) {
    if (q_len[r] < 0 || kv_len[r] < 1) return cudaErrorInvalidValue;
    tab.q_off[r] = q_off[r];
    tab.q_len[r] = q_len[r];
    tab.kv_off[r] = kv_off[r];
    tab.kv_len[r] = kv_len[r];
    tab.tile_start[r + 1] = tab.tile_start[r] + (q_len[r] + rows_per_block - 1) / rows_per_block;
    q_rows = std::max(q_rows, q_off[r] + q_len[r]);
    kv_rows = std::max(kv_rows, kv_off[r] + kv_len[r]);
  }
  return d == 128 ? launch<128>(Q, K, V, O, heads, q_rs, kv_rs, o_rs, tab, q_rows, kv_rows, stream, osc, v_rs)
                  : launch<64>(Q, K, V, O, heads, q_rs, kv_rs, o_rs, tab, q_rows, kv_rows, stream, osc, v_rs);
}

cudaError_t attention_tc(const void* Q, const void* K, const void* V, void* O, int heads, int d,
                         int q_rs, int kv_rs, int o_rs, const int* seq_off, const int* seq_len,
                         int nreq, int num_sms, cudaStream_t stream, const OScatter* scatter, int v_rs) {
  (void)num_sms;
  for (int r = 0; r < nreq; ++r)
    if (seq_len[r] < 1) return cudaErrorInvalidValue;
  return attention_tc_segments(Q, K, V, O, heads, d, q_rs, kv_rs, o_rs, seq_off, seq_len, seq_off, seq_len, nreq,
                               stream, scatter, v_rs);
}

}  // namespace gs

extern "C" int gs_debug_attention_ctatime(unsigned long long* host, size_t n) {
  if (!host || n > sizeof(gs::g_attn_ctatime) / 8) return -1;
  return cudaMemcpyFromSymbol(host, gs::g_attn_ctatime, n * 8) == cudaSuccess ? 0 : -4;
}

extern "C" int gs_debug_attention_trace(unsigned long long* host, size_t n) {
  if (!host || n > sizeof(gs::g_attn_trace) / 8) return -1;
  return cudaMemcpyFromSymbol(host, gs::g_attn_trace, n * 8) == cudaSuccess ? 0 : -4;
}
