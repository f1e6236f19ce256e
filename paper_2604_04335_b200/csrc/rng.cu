// Counter-based generator for synthetic weights and latent noise on the device.
// Same definition as DESIGN.md "Input recipe" (implemented independently from the numpy
// generator in synth/rng.py; tests/test_gpu_parity.py checks the two bitwise):
//   h = splitmix64(seed ^ (tensor_id << 40) ^ idx);  u = ((h >> 40) - 2^23) * 2^-23
//   bf16 weight = RNE(fp32(u * scale)); gain = RNE(fp32(1 + fp32(0.1 u))); fp32 = fp32(u * s)
//   noise z_i = fp32((u_{4i} + u_{4i+1} + u_{4i+2} + u_{4i+3}) * sqrt(3/4)) (fp64 sum)
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.h"

namespace gs {
namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ float unif(uint64_t key, uint64_t idx) {
  const uint64_t h = mix64(key ^ idx);
  const int top = static_cast<int>(h >> 40) - (1 << 23);
  return __fmul_rn(static_cast<float>(top), 1.1920928955078125e-07f);  // exact
}

__global__ void rng_fill_kernel(void* out, long long n, uint64_t key, int kind, float scale) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const float u = unif(key, static_cast<uint64_t>(i));
    if (kind == RNG_BF16_SCALED) {
      static_cast<__nv_bfloat16*>(out)[i] = __float2bfloat16_rn(__fmul_rn(u, scale));
    } else if (kind == RNG_BF16_GAIN) {
      static_cast<__nv_bfloat16*>(out)[i] = __float2bfloat16_rn(__fadd_rn(1.0f, __fmul_rn(u, 0.1f)));
    } else {
      static_cast<float*>(out)[i] = __fmul_rn(u, scale);
    }
  }
}

__global__ void rng_noise_kernel(float* out, long long first, long long n, uint64_t key) {
  const double c = 0.8660254037844386;  // sqrt(3/4), correctly rounded fp64
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const uint64_t g = static_cast<uint64_t>(first + i) * 4;
    const double s = ((double)unif(key, g) + (double)unif(key, g + 1)) +
                     ((double)unif(key, g + 2) + (double)unif(key, g + 3));  // exact
    out[i] = __double2float_rn(__dmul_rn(s, c));
  }
}
__global__ void rng_normal_bf16_kernel(__nv_bfloat16* out, long long n, uint64_t key) {
  const double c = 0.8660254037844386;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const uint64_t g = static_cast<uint64_t>(i) * 4;
    const double s = ((double)unif(key, g) + (double)unif(key, g + 1)) +
                     ((double)unif(key, g + 2) + (double)unif(key, g + 3));
    out[i] = __float2bfloat16_rn(__double2float_rn(__dmul_rn(s, c)));
  }
}
}  // namespace

cudaError_t rng_normal_bf16(__nv_bfloat16* out, long long n, uint64_t seed, uint32_t tensor_id,
                            cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  const uint64_t key = seed ^ (static_cast<uint64_t>(tensor_id) << 40);
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  rng_normal_bf16_kernel<<<static_cast<int>(blocks), 256, 0, stream>>>(out, n, key);
  return cudaGetLastError();
}

cudaError_t rng_fill(void* out, long long n, uint64_t seed, uint32_t tensor_id, int kind,
                     float scale, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  const uint64_t key = seed ^ (static_cast<uint64_t>(tensor_id) << 40);
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  rng_fill_kernel<<<static_cast<int>(blocks), 256, 0, stream>>>(out, n, key, kind, scale);
  return cudaGetLastError();
}

cudaError_t rng_noise(float* out, long long tok_lo, long long ntok, int channels, uint64_t seed,
                      cudaStream_t stream) {
  const long long n = ntok * channels;
  if (n <= 0) return cudaSuccess;
  const uint64_t key = seed;  // tensor_id 0
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  rng_noise_kernel<<<static_cast<int>(blocks), 256, 0, stream>>>(out, tok_lo * channels, n, key);
  return cudaGetLastError();
}

}  // namespace gs
