// Microbenchmark: cycles per tcgen05.mma (kind::f16, bf16 in, fp32 acc) for SS / TS operand
// modes and N in {64,128,256}, issued back to back by one thread into one TMEM accumulator.
// Operands are whatever is in smem/TMEM (values irrelevant).  One CTA per SM, grid = #SMs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2604_04335_b200/csrc umma_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace gs;

template <int MODE, int N>  // MODE 0 = SS, 1 = TS (A from TMEM)
__global__ void __launch_bounds__(128, 1) bench(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 32) {
    constexpr uint32_t idesc = idesc_bf16(128, N, 0, 0);
    const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 65536);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        if (MODE == 0)
          mma_ss(tmem + 256, sdesc_sw128(sa + kk * 32, 16, 1024), sdesc_sw128(sb + kk * 32, 16, 1024), idesc, 1);
        else
          mma_ts(tmem + 256, tmem + kk * 8, sdesc_sw128(sb + kk * 32, 16, 1024), idesc, 1);
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int MODE, int N>
void run(const char* name) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d;
  cudaMalloc(&d, sms * 8);
  const int smem = 160 * 1024;
  cudaFuncSetAttribute(bench<MODE, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  bench<MODE, N><<<sms, 128, smem>>>(iters, d);
  bench<MODE, N><<<sms, 128, smem>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[256];
  cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  avg /= sms;
  const double per = avg / (iters * 4.0);
  const double ideal = 128.0 * N / 256.0;
  printf("%-10s N=%3d: %7.1f cycles/MMA (ideal %5.1f) -> %5.1f%%  %s\n", name, N, per, ideal, 100 * ideal / per,
         cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<0, 64>("SS");
  run<0, 128>("SS");
  run<0, 256>("SS");
  run<1, 64>("TS");
  run<1, 128>("TS");
  run<1, 256>("TS");
  return 0;
}
