// tcgen05 GEMM for the DiT linear layers:
//   C[M,N] = A[M,K] . W[N,K]^T, bf16 operands, fp32 accumulation in TMEM, fused epilogues
//   (bias; GELU-tanh; fp32 gated residual x += g (.) (acc + b); Euler z += dsig (acc + b)).
//
// Design (B200-first):
//   * persistent kernel, one CTA per SM, static tile schedule (tile t = blockIdx.x + i*grid);
//   * warp 0: TMA producer (128B-swizzled K-major tiles, 4-stage mbarrier ring);
//   * warp 1: TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=256, K=16);
//   * warps 2..5: epilogue (tcgen05.ld 32x32b -> registers -> fused epilogue -> global);
//   * two TMEM accumulators (2 x 256 columns) so the epilogue of tile i overlaps the
//     main loop of tile i+1.
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
template <int BN>
struct GCfg {
  static constexpr int STAGES = BN == 256 ? 6 : 7;
  static constexpr int B_BYTES = (BN / 2) * BK * 2;  // this CTA's half of the W tile
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

__device__ __forceinline__ float gelu_tanh_f(float u) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  return 0.5f * u * (1.0f + tanh_approx(k0 * (u + k1 * u * u * u)));
}

template <int EPI>
__device__ __forceinline__ void epilogue_chunk(const uint32_t (&r)[32], int row, int col0,
                                               const EpiParams& ep) {
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
  if constexpr (EPI == EPI_BF16 || EPI == EPI_GELU_BF16) {
    uint32_t pk[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      float a = v[2 * i], b = v[2 * i + 1];
      if constexpr (EPI == EPI_GELU_BF16) {
        a = gelu_tanh_f(a);
        b = gelu_tanh_f(b);
      }
      pk[i] = pack_bf16x2(a, b);
    }
    uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(ep.out) +
                                          static_cast<size_t>(row) * ep.ldo + col0);
#pragma unroll
    for (int q = 0; q < 4; ++q) dst[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
  } else if constexpr (EPI == EPI_F32) {
    float4* dst = reinterpret_cast<float4*>(static_cast<float*>(ep.out) +
                                            static_cast<size_t>(row) * ep.ldo + col0);
#pragma unroll
    for (int q = 0; q < 8; ++q) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  } else if constexpr (EPI == EPI_RESID_F32) {
    const int req = ep.row_req[row];
    const float4* ga = reinterpret_cast<const float4*>(ep.gate_a + col0);
    const float4* gb =
        reinterpret_cast<const float4*>(ep.gate_b + static_cast<size_t>(req) * ep.gate_b_stride + col0);
    float4* dst = reinterpret_cast<float4*>(static_cast<float*>(ep.out) +
                                            static_cast<size_t>(row) * ep.ldo + col0);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float4 a = __ldg(ga + q), b = __ldg(gb + q), x = dst[q];
      x.x += (a.x + b.x) * v[4 * q + 0];
      x.y += (a.y + b.y) * v[4 * q + 1];
      x.z += (a.z + b.z) * v[4 * q + 2];
      x.w += (a.w + b.w) * v[4 * q + 3];
      dst[q] = x;
    }
  } else if constexpr (EPI == EPI_ADD_F32) {
    float4* dst = reinterpret_cast<float4*>(static_cast<float*>(ep.out) +
                                            static_cast<size_t>(row) * ep.ldo + col0);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float4 x = dst[q];
      x.x += v[4 * q + 0];
      x.y += v[4 * q + 1];
      x.z += v[4 * q + 2];
      x.w += v[4 * q + 3];
      dst[q] = x;
    }
  } else if constexpr (EPI == EPI_EULER_F32) {
    const float ds = ep.dsig[ep.row_req[row]];
    float4* dst = reinterpret_cast<float4*>(static_cast<float*>(ep.out) +
                                            static_cast<size_t>(row) * ep.ldo + col0);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float4 x = dst[q];
      x.x += ds * v[4 * q + 0];
      x.y += ds * v[4 * q + 1];
      x.z += ds * v[4 * q + 2];
      x.w += ds * v[4 * q + 3];
      dst[q] = x;
    }
  }
}

// Per-FLOP rate of 192-wide relative to 256-wide pair tiles (kbench at large grids: c4 sp1 qkv
// 1223 vs 1494, c4 sp8 qkv 1314 vs 1513 TFLOP/s; profiles/r01_notes.md).
constexpr double kNarrowRate = 0.85;

// Tile rasterisation: bands of GROUP_M M-tiles, N-major inside a band, so the ~148 tiles in
// flight cover a GROUP_M x (148 / GROUP_M) block whose A and W panels stay resident in L2.
constexpr int GROUP_M = 16;
__device__ __forceinline__ void tile_coords(int t, int num_m, int num_n, int& mb, int& nb) {
  const int per_group = GROUP_M * num_n;
  const int g = t / per_group, r = t - g * per_group;
  const int m0 = g * GROUP_M;
  const int gm = min(GROUP_M, num_m - m0);
  mb = m0 + r % gm;
  nb = r / gm;
}

template <int EPI, int BN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   int M, int N, int K, const __grid_constant__ EpiParams ep) {
  constexpr int STAGES = GCfg<BN>::STAGES, STAGE_BYTES = GCfg<BN>::STAGE_BYTES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* full = bars;                     // [STAGES] (leader's are used: both CTAs' bytes)
  uint64_t* empty = bars + STAGES;           // [STAGES] per CTA (multicast commit)
  uint64_t* tfull = bars + 2 * STAGES;       // [2] per CTA (multicast commit)
  uint64_t* tempty = bars + 2 * STAGES + 2;  // [2] leader's: 4 epilogue warps x 2 CTAs
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);

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
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
  }
  if (warp == 1) tmem_alloc_2sm(tmem_slot, TMEM_COLS);
  tc_fence_before();
  cluster_sync();  // barriers of both CTAs initialised before any remote arrive / TMA
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // producer (both CTAs): this CTA's A rows and W half, bytes counted by the leader
      int stage = 0;
      uint32_t phase = 0;
      for (int t = pair; t < num_tiles; t += npairs) {
        int mb, nb;
        tile_coords(t, num_m, num_n, mb, nb);
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
    // epilogue (both CTAs): warps 2..5 -> TMEM lane quarter (warp % 4) of this CTA's 128 rows
    const int quarter = warp & 3;
    const uint32_t tempty_leader = mapa_shared(smem_u32(&tempty[0]), 0);
    int it = 0;
    for (int t = pair; t < num_tiles; t += npairs, ++it) {
      int mb, nb;
      tile_coords(t, num_m, num_n, mb, nb);
      const int as = it & 1;
      const uint32_t aphase = (it >> 1) & 1;
      mbar_wait(&tfull[as], aphase);
      tc_fence_after();
      const int row = mb * PM + rank * BM + quarter * 32 + lane;
      const uint32_t tbase = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + as * BN;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        const int col0 = nb * BN + c * 32;
        if (col0 >= N) break;  // warp-uniform
        uint32_t r[32];
        GS_TMEM_LD32(tbase + c * 32, r);
        tmem_ld_wait();
        if (row < M) epilogue_chunk<EPI>(r, row, col0, ep);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_leader + as * 8);
    }
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
  CUtensorMap ta, tb;
  if (!make_tma_2d_bf16(&ta, A, K, M, static_cast<uint64_t>(lda) * 2, BK, BM)) return cudaErrorInvalidValue;
  if (!make_tma_2d_bf16(&tb, W, K, N, static_cast<uint64_t>(ldw) * 2, BK, BN / 2)) return cudaErrorInvalidValue;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tc_kernel<EPI, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         GCfg<BN>::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int tiles = ((M + PM - 1) / PM) * ((N + BN - 1) / BN);
  const int pairs = tiles < num_sms / 2 ? tiles : num_sms / 2;
  const int grid = 2 * pairs;  // clusters of 2 (CTA pairs on one TPC)
  gemm_tc_kernel<EPI, BN><<<grid, THREADS, GCfg<BN>::SMEM_BYTES, stream>>>(ta, tb, M, N, K, ep);
  return cudaGetLastError();
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
