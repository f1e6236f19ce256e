// Softmax inner-loop instruction mix per SMSP: does F2FP (bf16x2 pack) share the MUFU pipe?
// KIND 0: 2 ex2 per pair; 1: F2FP only; 2: 2 ex2 + F2FP; 3: 2 ex2 + F2FP + FADD2;
// 4: 2 ex2 + integer RNE bf16 pack (no F2FP); 5: FADD2 only.  W warps per SMSP.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint32_t f2fp(float lo, float hi) {
  uint32_t r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo)); return r; }
__device__ __forceinline__ uint32_t ipack(float lo, float hi) {  // RNE for finite positives
  uint32_t a = __float_as_uint(lo), b = __float_as_uint(hi);
  a += 0x7FFFu + ((a >> 16) & 1u);
  b += 0x7FFFu + ((b >> 16) & 1u);
  return __byte_perm(a, b, 0x7632);
}
template <int KIND>
__global__ void k(uint32_t* out, int iters) {
  float a[16];
  uint32_t acc = 0;
  float2 s = make_float2(0.f, 0.f);
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = -0.001f * (threadIdx.x + i);
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      float x = a[i], y = a[i + 1];
      if (KIND == 0 || KIND == 2 || KIND == 3 || KIND == 4) { x = ex2(x); y = ex2(y); }
      if (KIND == 1 || KIND == 2 || KIND == 3) acc ^= f2fp(x, y);
      if (KIND == 4) acc ^= ipack(x, y);
      if (KIND == 3 || KIND == 5) s = __fadd2_rn(s, make_float2(x, y));
      a[i] = x * 0.5f + (KIND == 1 ? 0.001f : 0.f);
      a[i + 1] = y;
      if (KIND == 1 || KIND == 5) { a[i] = __uint_as_float(__float_as_uint(a[i]) ^ (acc & 1)); }
    }
  }
  const long long t1 = clock64();
  float t = s.x + s.y;
#pragma unroll
  for (int i = 0; i < 16; ++i) t += a[i];
  if (t == 12345.f || acc == 0x12345678u) out[0] = acc;
  if (threadIdx.x == 0) out[1 + blockIdx.x] = uint32_t(t1 - t0);
}
template <int KIND> void run(uint32_t* d, const char* name) {
  for (int w = 1; w <= 4; w *= 2) {
    const int iters = 4000;
    k<KIND><<<148, 128 * w>>>(d, iters);
    cudaDeviceSynchronize();
    k<KIND><<<148, 128 * w>>>(d, iters);
    cudaDeviceSynchronize();
    uint32_t h[2];
    cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("%-28s warps/SMSP %d: %.2f cycles per pair per warp\n", name, w, double(h[1]) / (iters * 8.0 * w));
  }
}
int main() {
  uint32_t* d; cudaMalloc(&d, 4096 * 4);
  run<0>(d, "2 ex2");
  run<1>(d, "F2FP");
  run<2>(d, "2 ex2 + F2FP");
  run<3>(d, "2 ex2 + F2FP + FADD2");
  run<4>(d, "2 ex2 + int pack");
  run<5>(d, "FADD2");
  return 0;
}
