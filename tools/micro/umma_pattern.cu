// Microbenchmark of the attention MMA pattern: per "tile" S0 = SS N128 (8 x K16) -> cols [0,128),
// S1 -> [128,256), PV0 = TS (A = cols [0,64) of S0 region) -> O0 [256,384), PV1 -> O1 [384,512).
// VAR 0: no commits; 1: 4 commits per tile (like the kernel); 2: kernel order
// PV0_j, S0_j+1, PV1_j, S1_j+1 without commits; 3: like 2 with commits.
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace gs;

template <int VAR>
__global__ void __launch_bounds__(128, 1) bench(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[5];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { for (int i = 0; i < 5; ++i) mbar_init(&bar[i], 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 32) {
    constexpr uint32_t idesc_s = idesc_bf16(128, 128, 0, 0);
    constexpr uint32_t idesc_o = idesc_bf16(128, 128, 0, 1);
    const uint32_t sq = smem_u32(smem), sk = smem_u32(smem + 65536), sv = smem_u32(smem + 98304);
    auto S = [&](int w) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
        mma_ss(tmem + w * 128, sdesc_sw128(sq + w * 32768 + off, 16, 1024), sdesc_sw128(sk + off, 16, 1024), idesc_s, kk > 0);
      }
    };
    auto PV = [&](int w) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        mma_ts(tmem + 256 + w * 128, tmem + w * 128 + kk * 8, sdesc_sw128(sv + kk * 2048, 16384, 1024), idesc_o, 1);
    };
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (VAR < 2) {
        S(0); if (VAR & 1) mma_commit(&bar[0]);
        S(1); if (VAR & 1) mma_commit(&bar[1]);
        PV(0); if (VAR & 1) mma_commit(&bar[2]);
        PV(1); if (VAR & 1) mma_commit(&bar[3]);
      } else {
        PV(0); S(0); if (VAR & 1) mma_commit(&bar[0]);
        PV(1); if (VAR & 1) mma_commit(&bar[2]);
        S(1); if (VAR & 1) { mma_commit(&bar[1]); mma_commit(&bar[3]); }
      }
    }
    mma_commit(&bar[4]);
    mbar_wait(&bar[4], 0);
    const long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int VAR>
void run() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d;
  cudaMalloc(&d, sms * 8);
  const int smem = 160 * 1024;
  cudaFuncSetAttribute(bench<VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 1000;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  bench<VAR><<<sms, 128, smem>>>(iters, d);
  cudaEventRecord(a);
  bench<VAR><<<sms, 128, smem>>>(iters, d);
  cudaEventRecord(b);
  cudaError_t e = cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double flops = 4.0 * 2 * 128 * 128 * 128 * iters * sms;
  printf("VAR %d: %.3f ms  %.1f TFLOP/s %s\n", VAR, ms, flops / ms / 1e9, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<0>(); run<1>(); run<2>(); run<3>();
  return 0;
}
