// Packed exp2 on the MUFU pipe: ex2.approx.f32 vs ex2.approx.f16x2 vs ex2.approx.ftz.bf16x2 --
// warp-instructions per clock per SMSP and exp2 results (elements) per clock per SMSP.
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
template <int KIND>
__global__ void k(float* out, int iters) {
  unsigned a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const float f = -0.001f * (threadIdx.x + i);
    if (KIND == 0) a[i] = __float_as_uint(f);
    else if (KIND == 1) { __half2 h = __floats2half2_rn(f, f * 0.5f); a[i] = *reinterpret_cast<unsigned*>(&h); }
    else { __nv_bfloat162 h = __floats2bfloat162_rn(f, f * 0.5f); a[i] = *reinterpret_cast<unsigned*>(&h); }
  }
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (KIND == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+r"(a[i]));
      else if (KIND == 1) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a[i]));
      else asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a[i]));
    }
  }
  const long long t1 = clock64();
  unsigned s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s ^= a[i];
  if (s == 12345u) out[0] = 1.f;
  if (threadIdx.x == 0) out[1 + blockIdx.x] = float(t1 - t0);
}
int main() {
  float* d; cudaMalloc(&d, 4096 * 4);
  const char* nm[3] = {"ex2.f32     ", "ex2.f16x2   ", "ex2.bf16x2  "};
  for (int kind = 0; kind < 3; ++kind)
    for (int warps = 8; warps <= 16; warps *= 2) {
      const int iters = 2000;
      for (int rep = 0; rep < 2; ++rep) {
        if (kind == 0) k<0><<<148, warps * 32>>>(d, iters);
        else if (kind == 1) k<1><<<148, warps * 32>>>(d, iters);
        else k<2><<<148, warps * 32>>>(d, iters);
        cudaDeviceSynchronize();
      }
      float h[2]; cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
      const double instr = double(iters) * 16 * (warps / 4);
      const double elems = instr * 32 * (kind == 0 ? 1 : 2);
      printf("%s warps/SM %2d: %.2f cycles per warp-instr per SMSP, %.2f exp2 results/clk/SMSP\n", nm[kind], warps,
             h[1] / instr, elems / h[1]);
    }
  return 0;
}
