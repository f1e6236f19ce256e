// In-situ MMA cost of the v5 attention pattern (profiles/r01_notes.md r01z): the pair MMA pattern of
// one KV tile for two Q tiles (PV as TS, the v5 kernel) with and without 8 "softmax" warps per CTA
// doing the v5 softmax's TMEM traffic per tile (tcgen05.ld of 128 S columns, tcgen05.st of 64 P
// columns per row) -- does TMEM traffic slow the MMAs from 64 to the ~78 cycles seen in the kernel?
// (Derived from attn_pv_smem_bench.cu; MODE 1 there = P in shared memory.)
//
// CTA pairs (cta_group::2, M = 256), the leader's thread 32 issues per iteration the attention MMA
// pattern of one KV tile for two Q tiles: PV0, S0, PV1, S1 (8 x K16 MMAs each, 4 commits), with
//   MODE 0: PV as TS (A = P in TMEM, the v5 kernel);
//   MODE 1: PV as SS (A = P in shared memory, K-major 128B swizzle like Q);
// and WR = 1 adds 8 "softmax" warps per CTA storing 64 KB of P per iteration (st.shared.v4) into the
// P buffers, paced by the issuer (one iteration of stores per issued iteration).  No data
// dependencies: this measures throughput of the mix.  Reported: cycles per iteration (tile pair)
// on the leader, ideal 2048 (32 MMAs x 64 cycles).
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace gs;

constexpr int Q_OFF = 0, K_OFF = 65536, V_OFF = 81920, P_OFF = 98304, SMEM = 98304 + 65536 + 1024;

template <int MODE, int WR>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1) bench(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[5];
  __shared__ uint32_t slot;
  __shared__ volatile int progress;  // iterations issued by the leader's issuer (pacing for the writers)
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    for (int i = 0; i < 5; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
    progress = 0;
  }
  if (warp == 0) tmem_alloc_2sm(&slot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 32 && rank == 0) {
    constexpr uint32_t idesc_s = idesc_bf16(256, 128, 0, 0);
    constexpr uint32_t idesc_o = idesc_bf16(256, 128, 0, 1);
    const uint32_t sq = smem_u32(smem + Q_OFF), sk = smem_u32(smem + K_OFF), sv = smem_u32(smem + V_OFF);
    const uint32_t sp = smem_u32(smem + P_OFF);
    auto S = [&](int w) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t qoff = (kk >> 2) * 16384 + (kk & 3) * 32;
        const uint32_t koff = (kk >> 2) * 8192 + (kk & 3) * 32;
        mma_ss_2sm(tmem + w * 128, sdesc_sw128(sq + w * 32768 + qoff, 16, 1024), sdesc_sw128(sk + koff, 16, 1024),
                   idesc_s, kk > 0);
      }
    };
    auto PV = [&](int w) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint64_t vb = sdesc_sw128(sv + kk * 2048, 16384, 1024);
        if (MODE == 0) {
          mma_ts_2sm(tmem + 256 + w * 128, tmem + w * 128 + kk * 8, vb, idesc_o, 1);
        } else {
          const uint32_t poff = (kk >> 2) * 16384 + (kk & 3) * 32;
          mma_ss_2sm(tmem + 256 + w * 128, sdesc_sw128(sp + w * 32768 + poff, 16, 1024), vb, idesc_o, 1);
        }
      }
    };
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      PV(0);
      S(0);
      mma_commit_2sm_mc(&bar[0], 0x3);
      PV(1);
      mma_commit_2sm_mc(&bar[2], 0x3);
      S(1);
      mma_commit_2sm_mc(&bar[1], 0x3);
      mma_commit_2sm_mc(&bar[3], 0x3);
      progress = i + 1;
    }
    mma_commit_2sm_mc(&bar[4], 0x3);
    mbar_wait(&bar[4], 0);
    const long long t1 = clock64();
    out[blockIdx.x / 2] = t1 - t0;
  } else if (threadIdx.x == 32) {
    mbar_wait(&bar[4], 0);
  } else if (WR && warp >= 4) {
    // softmax warps 4..11 (quarter = warp & 3, group = (warp >> 2) - 1; warps 0 / 1 hold the TMEM
    // allocator and the issuer, and tcgen05.ld/st are warp-collective): per iteration load its 128 S columns
    // and store 64 columns of "P" over them, paced on the leader's issue counter (DSMEM)
    const uint32_t prog = mapa_shared(smem_u32((const void*)&progress), 0);
    const uint32_t tS = tmem + ((uint32_t)((warp & 3) * 32) << 16) + ((warp >> 2) - 1) * 128;
    uint32_t acc = 0;
    for (int i = 0; i < iters; ++i) {
      for (;;) {
        int p;
        asm volatile("ld.volatile.shared::cluster.u32 %0, [%1];" : "=r"(p) : "r"(prog) : "memory");
        if (p + 2 >= i) break;
      }
      uint32_t v[128];
      GS_TMEM_LD32(tS + 0, (*reinterpret_cast<uint32_t(*)[32]>(v + 0)));
      GS_TMEM_LD32(tS + 32, (*reinterpret_cast<uint32_t(*)[32]>(v + 32)));
      GS_TMEM_LD32(tS + 64, (*reinterpret_cast<uint32_t(*)[32]>(v + 64)));
      GS_TMEM_LD32(tS + 96, (*reinterpret_cast<uint32_t(*)[32]>(v + 96)));
      tmem_ld_wait();
      uint32_t pk[16];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
#pragma unroll
        for (int k = 0; k < 16; ++k) pk[k] = v[32 * c + 2 * k] ^ v[32 * c + 2 * k + 1];
        GS_TMEM_ST16(tS + c * 16, pk);
      }
      tmem_st_wait();
      acc += pk[0];
    }
    if (acc == 0x12345678u) out[0] = acc;
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc_2sm(tmem, 512);
  }
}

template <int MODE, int WR>
void run() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(bench<MODE, WR>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  const int iters = 2000;
  bench<MODE, WR><<<148, 384, SMEM>>>(iters, d);
  bench<MODE, WR><<<148, 384, SMEM>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[74];
  cudaMemcpy(h, d, 74 * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 74; ++i) avg += h[i];
  avg /= 74;
  const double per = avg / iters;
  printf("PV %s, softmax TMEM ld/st %s: %7.1f cycles per tile pair (ideal 2048) -> %5.1f%% of the MMA floor  %s\n",
         MODE == 0 ? "TS" : "SS", WR ? "on " : "off", per, 100.0 * 2048 / per, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<0, 0>();
  run<0, 1>();
  return 0;
}
