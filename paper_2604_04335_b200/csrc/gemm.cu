// tcgen05 GEMM for the DiT linear layers:
//   C[M,N] = A[M,K] . W[N,K]^T, bf16 operands, fp32 accumulation in TMEM, fused epilogues
//   (bias; GELU-tanh; fp32 gated residual x += g (.) (acc + b); Euler z += dsig (acc + b)).
//
// Design (B200-first):
//   * persistent CTA pairs (cta_group::2), static tile schedule (tile t = pair + i*npairs);
//   * warp 0: TMA producer (128B-swizzled K-major tiles, 5-7-stage mbarrier ring);
//   * warp 1: TMEM allocator + single-thread tcgen05.mma issuer (leader CTA, M=256, N=BN, K=16);
//   * warps 2..5: epilogue (tcgen05.ld 32x32b -> registers -> fused epilogue -> global; fp32
//     read-modify-write epilogues stream x through shared memory by TMA load / store);
//   * two TMEM accumulators (2 x BN columns) so the epilogue of tile i overlaps the
//     main loop of tile i+1;
//   * tiles in bands of GROUP_M M-tiles (L2 reuse of A / W panels); griddepcontrol.wait after the
//     setup (programmatic dependent launch).
// Bit-exactness across M (SURVEY.md §8(a) invariant 1): no split-K, no atomics, the same
// MMA shape and K order for every tile, each output row depends only on its own A row.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <cmath>
#include <cstdlib>

#include "kernels.h"
#include "ptx.cuh"
#include "tma.h"

namespace gs {

namespace {
// CTA-pair (cta_group::2) tiles: the pair computes 256 x 256 outputs with M=256 N=256 K=16 MMAs
// issued by the leader CTA; each CTA stages its 128 A rows and its 128-row half of W per stage,
// and holds its 128 output rows x 256 fp32 columns in its own TMEM.
// BN = 256 (default) or 192 (N % 192 == 0 and the 192-wide grid fills its waves enough better
// to pay for its ~15% lower per-FLOP rate: small-M grids such as config 3 at SP 4 / 8, where
// M = 4095 gives 96 256-wide tiles on 74 pairs).  Both issue
// M=256 K=16 MMAs over the same K order; the N width does not change any output element's
// accumulation (tests/test_gpu_kernels.py checks the two widths bit for bit), so the choice may
// depend on M without breaking SP / batch invariance.  (128-wide tiles were measured 35% slower
// per FLOP: 1.5x the L2 -> SM bytes; profiles/r01_notes.md.)
constexpr int BM = 128;                     // output rows per CTA (pair tile: 256)
constexpr int PM = 2 * BM;                  // pair tile rows
constexpr int BK = 64;
constexpr int A_BYTES = BM * BK * 2;        // 16 KB
constexpr int THREADS = 192;
constexpr uint32_t TMEM_COLS = 512;         // 2 accumulators x (up to) 256 columns
// Epilogues.  tcgen05.ld gives thread = row, 32 fp32 columns per load ("chunk").
//  * bf16 / fp32 outputs (write-only): each warp re-distributes its 32 rows x 32 columns through a
//    shared-memory transpose buffer so that 8 lanes cover one row's 32 columns and every global
//    store is a contiguous row segment.  Row pitch 36 floats (144 B): the float4 writes (lane =
//    row) and reads (8 lanes per row) are conflict-free per quarter-warp.
//  * fp32 read-modify-write (gated residual x, ungated residual, Euler latent z): the 32 x 32
//    chunk of x streams through a per-warp ring of XR_NB 4 KB shared-memory buffers by TMA
//    (128B-swizzled boxes, XR_LOOK chunks ahead), each thread updates its own row in place, and a
//    TMA store writes the chunk back.  No thread ever waits on a global load: the epilogue of a
//    short-K GEMM (config-2 O-proj, K = 1536) was latency-bound on its x loads at ~20 us per tile
//    against a ~6.5 us main loop (ncu: long-scoreboard stalls).
// The arithmetic per element is the same in both paths.
constexpr int EP_PITCH = 36;
constexpr int EP_WARP_BYTES = 32 * EP_PITCH * 4;
constexpr int EP_BYTES = 4 * EP_WARP_BYTES;  // 4 epilogue warps
constexpr int XR_NB = 4, XR_LOOK = 2;        // ring depth, load lookahead (chunks)
constexpr int XR_CHUNK = 32 * 32 * 4;        // 4 KB
constexpr int XR_BYTES = 4 * XR_NB * XR_CHUNK;
constexpr int BAR_BYTES = 1024;              // barriers + TMEM slot; keeps the ring 1024-aligned
template <int EPI>
constexpr bool kEpiReadsOut = EPI == EPI_RESID_F32 || EPI == EPI_ADD_F32 || EPI == EPI_EULER_F32;

template <int BN, bool RMW>
struct GCfg {
  static constexpr int STAGES = RMW ? 5 : (BN == 256 ? 6 : 7);
  static constexpr int B_BYTES = (BN / 2) * BK * 2;  // this CTA's half of the W tile
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + BAR_BYTES + (RMW ? XR_BYTES : EP_BYTES);
  static_assert(SMEM_BYTES <= 232448, "shared memory");
};

__device__ __forceinline__ float gelu_tanh_f(float u) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  return 0.5f * u * (1.0f + tanh_approx(k0 * (u + k1 * u * u * u)));
}

__device__ __forceinline__ void add4(float4& a, const float4& b) {
  a.x += b.x;
  a.y += b.y;
  a.z += b.z;
  a.w += b.w;
}

// Write-only epilogue of one 32 x 32 chunk of a warp's rows (row0 .. row0 + 31), columns
// col0 .. col0 + 31, through the warp's transpose buffer at shared address tw.
template <int EPI>
__device__ __forceinline__ void epilogue_chunk(uint32_t tw, const uint32_t (&r)[32], int row0, int col0, int M,
                                               const EpiParams& ep) {
  const int lane = threadIdx.x & 31;
  if (EPI == EPI_BF16 && ep.ssq != nullptr && col0 < ep.ssq_cols) {
    // this thread holds row row0 + lane's 32 columns: sum of (acc + bias)^2 in column order (two chains)
    float b[32];
    if (ep.bias != nullptr) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 braw = __ldg(reinterpret_cast<const uint4*>(ep.bias + col0) + q);
        const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&braw);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(b2[e]);
          b[8 * q + 2 * e] = f.x;
          b[8 * q + 2 * e + 1] = f.y;
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) b[i] = 0.f;
    }
    float s0 = 0.f, s1 = 0.f;
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      const float u0 = __uint_as_float(r[i]) + b[i], u1 = __uint_as_float(r[i + 1]) + b[i + 1];
      s0 = fmaf(u0, u0, s0);
      s1 = fmaf(u1, u1, s1);
    }
    const int row = row0 + lane;
    if (row < M) ep.ssq[static_cast<size_t>(row) * (ep.ssq_cols >> 5) + (col0 >> 5)] = s0 + s1;
  }
#pragma unroll
  for (int q = 0; q < 8; ++q)
    sts_v4(tw + (lane * EP_PITCH + 4 * q) * 4,
           make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]), __uint_as_float(r[4 * q + 2]),
                       __uint_as_float(r[4 * q + 3])));
  __syncwarp();
  const int rsub = lane >> 3, c4 = lane & 7;
  const int col = col0 + 4 * c4;
  float4 v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = lds_v4(tw + ((4 * i + rsub) * EP_PITCH + 4 * c4) * 4);
  __syncwarp();  // the buffer is rewritten by the next chunk
  if (ep.bias != nullptr) {
    const uint2 braw = __ldg(reinterpret_cast<const uint2*>(ep.bias + col));
    const float2 b01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&braw.x));
    const float2 b23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&braw.y));
    const float4 b = make_float4(b01.x, b01.y, b23.x, b23.y);
#pragma unroll
    for (int i = 0; i < 8; ++i) add4(v[i], b);
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int row = row0 + 4 * i + rsub;
    if (row >= M) continue;
    if constexpr (EPI == EPI_F32) {
      *reinterpret_cast<float4*>(static_cast<float*>(ep.out) + static_cast<size_t>(row) * ep.ldo + col) = v[i];
    } else {
      float4 f = v[i];
      if constexpr (EPI == EPI_GELU_BF16) {
        f.x = gelu_tanh_f(f.x);
        f.y = gelu_tanh_f(f.y);
        f.z = gelu_tanh_f(f.z);
        f.w = gelu_tanh_f(f.w);
      }
      *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(ep.out) + static_cast<size_t>(row) * ep.ldo + col) =
          make_uint2(pack_bf16x2(f.x, f.y), pack_bf16x2(f.z, f.w));
    }
  }
}

// Read-modify-write epilogue of one chunk: this thread's row lives in the 128B-swizzled 32 x 32
// fp32 box at shared address xb (16-byte unit j of row l at l * 128 + ((j ^ (l & 7)) << 4));
// updated in place for the TMA store.
template <int EPI>
__device__ __forceinline__ void rmw_chunk(uint32_t xb, const uint32_t (&r)[32], int col0, int req,
                                          const EpiParams& ep) {
  const int lane = threadIdx.x & 31;
  const uint32_t rowb = xb + lane * 128;
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
  if (ep.bias != nullptr) {
    const uint4* bp = reinterpret_cast<const uint4*>(ep.bias + col0);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 b = __ldg(bp + q);
      const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&b);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float2 f = __bfloat1622float2(b2[e]);
        v[q * 8 + 2 * e] += f.x;
        v[q * 8 + 2 * e + 1] += f.y;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const uint32_t addr = rowb + ((q ^ (lane & 7)) << 4);
    float4 x = lds_v4(addr);
    if constexpr (EPI == EPI_RESID_F32) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(ep.gate_a + col0) + q);
      const float4 b =
          __ldg(reinterpret_cast<const float4*>(ep.gate_b + static_cast<size_t>(req) * ep.gate_b_stride + col0) + q);
      x.x += (a.x + b.x) * v[4 * q + 0];
      x.y += (a.y + b.y) * v[4 * q + 1];
      x.z += (a.z + b.z) * v[4 * q + 2];
      x.w += (a.w + b.w) * v[4 * q + 3];
    } else if constexpr (EPI == EPI_ADD_F32) {
      x.x += v[4 * q + 0];
      x.y += v[4 * q + 1];
      x.z += v[4 * q + 2];
      x.w += v[4 * q + 3];
    } else {  // EPI_EULER_F32
      const float ds = ep.dsig[req];
      x.x += ds * v[4 * q + 0];
      x.y += ds * v[4 * q + 1];
      x.z += ds * v[4 * q + 2];
      x.w += ds * v[4 * q + 3];
    }
    sts_v4(addr, x);
  }
}

// Per-FLOP rate of 192-wide relative to 256-wide pair tiles (kbench at large grids: c4 sp1 qkv
// 1223 vs 1494, c4 sp8 qkv 1314 vs 1513 TFLOP/s; profiles/r01_notes.md).
constexpr double kNarrowRate = 0.85;

// Tile rasterisation: bands of GROUP_M M-tiles, N-major inside a band, so the ~148 tiles in
// flight cover a GROUP_M x (148 / GROUP_M) block whose A and W panels stay resident in L2.
constexpr int GROUP_M = 16;
__device__ __forceinline__ void tile_coords(int t, int num_m, int num_n, int group_m, int& mb, int& nb) {
  const int per_group = group_m * num_n;
  const int g = t / per_group, r = t - g * per_group;
  const int m0 = g * group_m;
  const int gm = min(group_m, num_m - m0);
  mb = m0 + r % gm;
  nb = r / gm;
}

template <int EPI, int BN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmX, int M, int N, int K,
                   const __grid_constant__ EpiParams ep) {
  constexpr bool RMW = kEpiReadsOut<EPI>;
  constexpr int STAGES = GCfg<BN, RMW>::STAGES, STAGE_BYTES = GCfg<BN, RMW>::STAGE_BYTES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* full = bars;                     // [STAGES] (leader's are used: both CTAs' bytes)
  uint64_t* empty = bars + STAGES;           // [STAGES] per CTA (multicast commit)
  uint64_t* tfull = bars + 2 * STAGES;       // [2] per CTA (multicast commit)
  uint64_t* tempty = bars + 2 * STAGES + 2;  // [2] leader's: 4 epilogue warps x 2 CTAs
  uint64_t* xfull = bars + 2 * STAGES + 4;   // [4 warps][XR_NB] (RMW epilogues)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4 + 4 * XR_NB);
  uint8_t* ep_smem = smem + STAGES * STAGE_BYTES + BAR_BYTES;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int num_m = (M + PM - 1) / PM, num_n = (N + BN - 1) / BN;
  const int num_tiles = num_m * num_n, num_k = K / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 2);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 8);
    }
    for (int s = 0; s < 4 * XR_NB; ++s) mbar_init(&xfull[s], 1);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    if constexpr (RMW) tma_prefetch(&tmX);
  }
  if (warp == 1) tmem_alloc_2sm(tmem_slot, TMEM_COLS);
  tc_fence_before();
  cluster_sync();  // barriers of both CTAs initialised before any remote arrive / TMA
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();  // the setup above overlaps the previous kernel's tail; global memory only from here
  pdl_launch_dependents();

  if (warp == 0) {
    if (lane == 0) {  // producer (both CTAs): this CTA's A rows and W half, bytes counted by the leader
      int stage = 0;
      uint32_t phase = 0;
      for (int t = pair; t < num_tiles; t += npairs) {
        int mb, nb;
        tile_coords(t, num_m, num_n, ep.group_m, mb, nb);
        for (int kb = 0; kb < num_k; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          mbar_arrive_expect_tx_cluster(mapa_shared(smem_u32(&full[stage]), 0), STAGE_BYTES);
          tma_load_2d_2sm(&tmA, &full[stage], sa, kb * BK, mb * PM + rank * BM);
          tma_load_2d_2sm(&tmB, &full[stage], sa + A_BYTES, kb * BK, nb * BN + rank * (BN / 2));
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {  // MMA issuer: leader CTA only
      constexpr uint32_t idesc = idesc_bf16(PM, BN, 0, 0);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = pair; t < num_tiles; t += npairs, ++it) {
        const int as = it & 1;
        const uint32_t aphase = (it >> 1) & 1;
        mbar_wait(&tempty[as], aphase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + as * BN;
        for (int kb = 0; kb < num_k; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t sb = sa + A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            mma_ss_2sm(d_tmem, sdesc_sw128(sa + kk * 32, 16, 1024), sdesc_sw128(sb + kk * 32, 16, 1024), idesc,
                       (kb | kk) != 0);
          mma_commit_2sm_mc(&empty[stage], 0x3);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit_2sm_mc(&tfull[as], 0x3);
      }
    }
  } else {
    // epilogue (both CTAs): warps 2..5 -> TMEM lane quarter (warp % 4) of this CTA's 128 rows.
    // TMEM loads run one 32-column chunk ahead of the global-memory work; the accumulator is
    // handed back to the MMA issuer as soon as its last chunk is in registers.
    const int quarter = warp & 3, we = warp - 2;
    const uint32_t tw = smem_u32(ep_smem) + we * EP_WARP_BYTES;              // write-only path
    const uint32_t ring = smem_u32(ep_smem) + we * XR_NB * XR_CHUNK;         // RMW path
    uint64_t* wxfull = xfull + we * XR_NB;
    const uint32_t tempty_leader = mapa_shared(smem_u32(&tempty[0]), 0);
    // RMW load cursor: the (tile, chunk) sequence this warp will consume, XR_LOOK chunks ahead.
    int lt = pair, lc = 0, lnch = 0, lcol = 0, lrow = 0;
    uint32_t nload = 0, ncons = 0;
    auto load_tile = [&]() {
      if (lt < num_tiles) {
        int mb, nb;
        tile_coords(lt, num_m, num_n, ep.group_m, mb, nb);
        lnch = min(BN, N - nb * BN) / 32;
        lcol = nb * BN;
        lrow = mb * PM + rank * BM + quarter * 32;
      }
    };
    auto issue_load = [&]() {  // next chunk of the cursor into ring slot nload % XR_NB
      if (lt >= num_tiles) return;
      if (lane == 0) {
        const int b = nload % XR_NB;
        // slot b last held chunk nload - XR_NB, whose store is older than the newest
        // XR_NB - XR_LOOK - 1 committed stores
        bulk_wait_group_read<XR_NB - XR_LOOK - 1>();
        mbar_arrive_expect_tx(&wxfull[b], XR_CHUNK);
        tma_load_2d(&tmX, &wxfull[b], ep_smem + (we * XR_NB + b) * XR_CHUNK, lcol + lc * 32, lrow);
      }
      ++nload;
      if (++lc == lnch) {
        lc = 0;
        lt += npairs;
        load_tile();
      }
    };
    if constexpr (RMW) {
      load_tile();
      for (int i = 0; i < XR_LOOK; ++i) issue_load();
    }
    auto do_chunk = [&](const uint32_t (&r)[32], int row0, int col0, int req) {
      if constexpr (RMW) {
        issue_load();
        const int b = ncons % XR_NB;
        mbar_wait(&wxfull[b], (ncons / XR_NB) & 1);
        ++ncons;
        const uint32_t xb = ring + b * XR_CHUNK;
        rmw_chunk<EPI>(xb, r, col0, req, ep);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&tmX, ep_smem + (we * XR_NB + b) * XR_CHUNK, col0, row0);
          bulk_commit_group();
        }
      } else {
        epilogue_chunk<EPI>(tw, r, row0, col0, M, ep);
      }
    };
    int it = 0;
    for (int t = pair; t < num_tiles; t += npairs, ++it) {
      int mb, nb;
      tile_coords(t, num_m, num_n, ep.group_m, mb, nb);
      const int as = it & 1;
      const uint32_t aphase = (it >> 1) & 1;
      mbar_wait(&tfull[as], aphase);
      tc_fence_after();
      const int row0 = mb * PM + rank * BM + quarter * 32;
      const uint32_t tbase = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + as * BN;
      const int nch = min(BN, N - nb * BN) / 32;  // N % 32 == 0
      int req = 0;
      if constexpr (EPI == EPI_RESID_F32 || EPI == EPI_EULER_F32)
        if (row0 + lane < M) req = __ldg(ep.row_req + row0 + lane);
      uint32_t ra[32], rb[32];
      GS_TMEM_LD32(tbase, ra);
#pragma unroll 1
      for (int c = 0; c < nch; c += 2) {
        GS_TMEM_LD_WAIT_REGS32(ra);
        if (c + 1 < nch) GS_TMEM_LD32(tbase + (c + 1) * 32, rb);
        if (c + 1 >= nch) {  // all of this accumulator is in registers
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(tempty_leader + as * 8);
        }
        do_chunk(ra, row0, nb * BN + c * 32, req);
        if (c + 1 < nch) {
          GS_TMEM_LD_WAIT_REGS32(rb);
          if (c + 2 < nch) GS_TMEM_LD32(tbase + (c + 2) * 32, ra);
          if (c + 2 >= nch) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(tempty_leader + as * 8);
          }
          do_chunk(rb, row0, nb * BN + (c + 1) * 32, req);
        }
      }
    }
    if constexpr (RMW)
      if (lane == 0) bulk_wait_group_all();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the peer may still read our smem / arrive on our barriers until here
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_2sm(tmem_base, TMEM_COLS);
  }
}

template <int EPI, int BN>
cudaError_t launch_bn(int M, int N, int K, const void* A, int lda, const void* W, int ldw,
                      const EpiParams& ep, int num_sms, cudaStream_t stream) {
  constexpr bool RMW = kEpiReadsOut<EPI>;
  CUtensorMap ta, tb, tx;
  if (!make_tma_2d_bf16(&ta, A, K, M, static_cast<uint64_t>(lda) * 2, BK, BM)) return cudaErrorInvalidValue;
  if (!make_tma_2d_bf16(&tb, W, K, N, static_cast<uint64_t>(ldw) * 2, BK, BN / 2)) return cudaErrorInvalidValue;
  if (RMW) {
    if (ep.ldo % 4 || (reinterpret_cast<uintptr_t>(ep.out) & 15)) return cudaErrorInvalidValue;
    if (!make_tma_2d_f32(&tx, ep.out, N, M, static_cast<uint64_t>(ep.ldo) * 4, 32, 32)) return cudaErrorInvalidValue;
  } else {
    tx = ta;  // unused
  }
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tc_kernel<EPI, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         GCfg<BN, RMW>::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int tiles = ((M + PM - 1) / PM) * ((N + BN - 1) / BN);
  const int pairs = tiles < num_sms / 2 ? tiles : num_sms / 2;
  const int grid = 2 * pairs;  // clusters of 2 (CTA pairs on one TPC)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = GCfg<BN, RMW>::SMEM_BYTES;
  cfg.stream = stream;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr.val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  static const int group_m = [] {
    const char* e = getenv("GS_GEMM_GROUP_M");  // development aid (A/B of the rasterisation band)
    const int g = e ? atoi(e) : GROUP_M;
    return g > 0 ? g : GROUP_M;
  }();
  EpiParams epg = ep;
  epg.group_m = group_m;
  return cudaLaunchKernelEx(&cfg, gemm_tc_kernel<EPI, BN>, ta, tb, tx, M, N, K, epg);
}

int pick_bn(int M, int N, int num_sms) {
  static const int env = [] {
    const char* e = getenv("GS_GEMM_BN");
    return e ? atoi(e) : 0;
  }();
  const int forced = g_gemm_bn_override.load(std::memory_order_relaxed);
  const int f = forced ? forced : env;
  if (f == 192 && N % 192 == 0) return 192;
  if (f == 256) return 256;
  if (N % 192) return 256;
  const double pairs = num_sms / 2;
  const double mt = (M + PM - 1) / PM;
  auto fill = [&](int bn) {  // fraction of the pair-slots x waves doing useful tiles
    const double tiles = mt * (N / bn);
    return tiles / (std::ceil(tiles / pairs) * pairs) * bn / 256.0 * (256.0 / bn);
  };
  return fill(192) * kNarrowRate > fill(256) ? 192 : 256;
}

template <int EPI>
cudaError_t launch(int M, int N, int K, const void* A, int lda, const void* W, int ldw,
                   const EpiParams& ep, int num_sms, cudaStream_t stream) {
  if (pick_bn(M, N, num_sms) == 192) return launch_bn<EPI, 192>(M, N, K, A, lda, W, ldw, ep, num_sms, stream);
  return launch_bn<EPI, 256>(M, N, K, A, lda, W, ldw, ep, num_sms, stream);
}
}  // namespace
std::atomic<int> g_gemm_bn_override{0};

cudaError_t gemm_bf16_tc(int epi, int M, int N, int K, const void* A, int lda, const void* W,
                         int ldw, const EpiParams& ep, int num_sms, cudaStream_t stream) {
  if (M <= 0 || N <= 0 || K <= 0 || K % BK != 0 || N % 32 != 0 || lda % 8 || ldw % 8)
    return cudaErrorInvalidValue;
  switch (epi) {
    case EPI_BF16: return launch<EPI_BF16>(M, N, K, A, lda, W, ldw, ep, num_sms, stream);
    case EPI_GELU_BF16: return launch<EPI_GELU_BF16>(M, N, K, A, lda, W, ldw, ep, num_sms, stream);
    case EPI_F32: return launch<EPI_F32>(M, N, K, A, lda, W, ldw, ep, num_sms, stream);
    case EPI_RESID_F32: return launch<EPI_RESID_F32>(M, N, K, A, lda, W, ldw, ep, num_sms, stream);
    case EPI_EULER_F32: return launch<EPI_EULER_F32>(M, N, K, A, lda, W, ldw, ep, num_sms, stream);
    case EPI_ADD_F32: return launch<EPI_ADD_F32>(M, N, K, A, lda, W, ldw, ep, num_sms, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace gs
