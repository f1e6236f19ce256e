// cycles per tcgen05.mma.cta_group::2 (M=256, N in {128,256}) issued back to back by the leader CTA.
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace gs;
template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) bench(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc_2sm(&slot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 32 && rank == 0) {
    constexpr uint32_t idesc = idesc_bf16(256, N, 0, 0);
    const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 65536);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        mma_ss_2sm(tmem, sdesc_sw128(sa + kk * 32, 16, 1024), sdesc_sw128(sb + kk * 32, 16, 1024), idesc, 1);
    }
    mma_commit_2sm_mc(&bar, 0x3);
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    out[blockIdx.x / 2] = t1 - t0;
  } else if (threadIdx.x == 32) {
    mbar_wait(&bar, 0);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) { tc_fence_after(); tmem_dealloc_2sm(tmem, 512); }
}
template <int N>
void run() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  const int smem = 160 * 1024;
  cudaFuncSetAttribute(bench<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  bench<N><<<148, 128, smem>>>(iters, d);
  bench<N><<<148, 128, smem>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[74];
  cudaMemcpy(h, d, 74 * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 74; ++i) avg += h[i];
  avg /= 74;
  const double per = avg / (iters * 4.0);
  const double ideal = 256.0 * N / 512.0;
  printf("2SM M256 N=%3d: %7.1f cycles/MMA (ideal %5.1f) -> %5.1f%%  %s\n", N, per, ideal, 100 * ideal / per, cudaGetErrorString(e));
}
int main() { run<128>(); run<256>(); return 0; }
// (appended) occupancy query
#include <cstdlib>
struct OccQuery {
  OccQuery() {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148);
    cfg.blockDim = dim3(192);
    int smems[3] = {160 * 1024, 197888, 227 * 1024};
    for (int i = 0; i < 3; ++i) {
      cfg.dynamicSmemBytes = smems[i];
      cudaLaunchAttribute attr;
      attr.id = cudaLaunchAttributeClusterDimension;
      attr.val.clusterDim.x = 2; attr.val.clusterDim.y = 1; attr.val.clusterDim.z = 1;
      cfg.attrs = &attr; cfg.numAttrs = 1;
      cudaFuncSetAttribute(bench<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smems[i]);
      int n = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, bench<256>, &cfg);
      printf("smem %d: max active clusters of 2 = %d (%s)\n", smems[i], n, cudaGetErrorString(e));
    }
  }
} g_occ;
