// MUFU.EX2 / FFMA2 throughput per SMSP: W warps per SMSP each issuing independent ops.
#include <cstdio>
#include <cuda_runtime.h>
template <int KIND>
__global__ void k(float* out, int iters) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = -0.001f * (threadIdx.x + i);
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (KIND == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      else if (KIND == 1) a[i] = fmaf(a[i], 0.999f, -0.001f);
    }
  }
  const long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == 12345.f) out[0] = s;
  if (threadIdx.x == 0) out[1 + blockIdx.x] = float(t1 - t0);
}
int main() {
  float* d; cudaMalloc(&d, 4096 * 4);
  for (int kind = 0; kind < 2; ++kind)
    for (int warps = 4; warps <= 32; warps *= 2) {
      const int iters = 2000;
      if (kind == 0) { k<0><<<148, warps * 32>>>(d, iters); cudaDeviceSynchronize(); k<0><<<148, warps * 32>>>(d, iters); }
      else { k<1><<<148, warps * 32>>>(d, iters); cudaDeviceSynchronize(); k<1><<<148, warps * 32>>>(d, iters); }
      cudaDeviceSynchronize();
      float h[2]; cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
      const double ops_per_smsp = double(iters) * 16 * (warps / 4) * 32;
      printf("%s warps/SM %2d: %.2f ops/clk/SMSP (%.1f cycles per warp-instr per SMSP)\n", kind == 0 ? "ex2 " : "ffma",
             warps, ops_per_smsp / h[1], h[1] / (iters * 16.0 * (warps / 4)));
    }
  return 0;
}
