// Element-wise kernels of the VAE decode stage (oracle: oracle/vae.py).
// HBM-bound: coalesced 16-byte accesses, fp32 math, bf16 storage (RNE).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "kernels.h"
#include "ptx.cuh"

namespace gs {
namespace {

// z[f, 2h + ph, 2w + pw, c] = lat[(f, h, w), c*4 + ph*2 + pw] * std[c] + mean[c]; one thread per
// output voxel writes its 64 padded channels (8 x 16 B).
__global__ void vae_unpatchify_kernel(const float* __restrict__ lat, int F, int Ht, int Wt,
                                      const float* __restrict__ mean, const float* __restrict__ stdv,
                                      __nv_bfloat16* __restrict__ z, int zc) {
  const long long nvox = static_cast<long long>(F) * 2 * Ht * 2 * Wt;
  const long long v = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (v >= nvox) return;
  const int W2 = 2 * Wt, H2 = 2 * Ht;
  const int x = static_cast<int>(v % W2), y = static_cast<int>((v / W2) % H2), f = static_cast<int>(v / (W2 * H2));
  const long long tok = (static_cast<long long>(f) * Ht + y / 2) * Wt + x / 2;
  const int sub = (y & 1) * 2 + (x & 1);
  const float* src = lat + tok * 64;
  uint32_t pk[32];
#pragma unroll
  for (int c = 0; c < 16; c += 2)
    pk[c / 2] = pack_bf16x2(__ldg(src + c * 4 + sub) * __ldg(stdv + c) + __ldg(mean + c),
                            __ldg(src + (c + 1) * 4 + sub) * __ldg(stdv + c + 1) + __ldg(mean + c + 1));
#pragma unroll
  for (int i = 8; i < 32; ++i) pk[i] = 0u;
  uint4* dst = reinterpret_cast<uint4*>(z + v * zc);
  for (int q = 0; q < zc / 8; ++q) dst[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
}

// One warp per voxel: lane l holds channels [8 l, 8 l + 8) of each 256-channel slice (Cp <= 512);
// input fp32 (the residual stream) or bf16.
template <bool F32>
__global__ void vae_rmsnorm_silu_kernel(const void* __restrict__ xin, long long nvox, int C, int Cp,
                                        const __nv_bfloat16* __restrict__ gamma, __nv_bfloat16* __restrict__ y) {
  const long long v = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (v >= nvox) return;
  float a[2][8];
  float ss = 0.f;
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int c0 = s * 256 + lane * 8;
    if (c0 < Cp) {
      float f[8];
      if (F32) {
        const float4* r4 = reinterpret_cast<const float4*>(static_cast<const float*>(xin) + v * Cp + c0);
        const float4 lo = r4[0], hi = r4[1];
        f[0] = lo.x; f[1] = lo.y; f[2] = lo.z; f[3] = lo.w; f[4] = hi.x; f[5] = hi.y; f[6] = hi.z; f[7] = hi.w;
      } else {
        const uint4 raw = *reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(xin) + v * Cp + c0);
        const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 t2 = __bfloat1622float2(h2[j]);
          f[2 * j] = t2.x;
          f[2 * j + 1] = t2.y;
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) a[s][j] = c0 + j < C ? f[j] : 0.f;
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) a[s][j] = 0.f;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) ss = fmaf(a[s][j], a[s][j], ss);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const float scale = sqrtf(static_cast<float>(C)) / fmaxf(sqrtf(ss), 1e-12f);
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int c0 = s * 256 + lane * 8;
    if (c0 >= Cp) continue;
    uint32_t pk[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float u[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = c0 + 2 * j + e;
        const float g = c < C ? __bfloat162float(gamma[c]) : 0.f;
        const float n = a[s][2 * j + e] * scale * g;
        u[e] = n / (1.0f + __expf(-n));
      }
      pk[j] = pack_bf16x2(u[0], u[1]);
    }
    *reinterpret_cast<uint4*>(y + v * Cp + c0) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
  }
}

// One thread per (output voxel, 8-channel chunk): fp32 (RNE) or bf16 in, bf16 out.
template <bool F32>
__global__ void vae_upsample2_kernel(const void* __restrict__ xin, int T, int H, int W, int Cp,
                                     __nv_bfloat16* __restrict__ y) {
  const int nch = Cp / 8;
  const long long total = static_cast<long long>(T) * 2 * H * 2 * W * nch;
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= total) return;
  const int ch = static_cast<int>(i % nch);
  const long long ov = i / nch;
  const int W2 = 2 * W, H2 = 2 * H;
  const int ox = static_cast<int>(ov % W2), oy = static_cast<int>((ov / W2) % H2);
  const long long t = ov / (static_cast<long long>(W2) * H2);
  const long long iv = (t * H + oy / 2) * W + ox / 2;
  if (F32) {
    const float4* src = reinterpret_cast<const float4*>(static_cast<const float*>(xin) + (iv * nch + ch) * 8);
    const float4 a = __ldg(src), b = __ldg(src + 1);
    reinterpret_cast<uint4*>(y)[ov * nch + ch] =
        make_uint4(pack_bf16x2(a.x, a.y), pack_bf16x2(a.z, a.w), pack_bf16x2(b.x, b.y), pack_bf16x2(b.z, b.w));
  } else {
    reinterpret_cast<uint4*>(y)[ov * nch + ch] = __ldg(static_cast<const uint4*>(xin) + iv * nch + ch);
  }
}

__global__ void vae_cast_bf16_kernel(const float4* __restrict__ x, long long n4, uint2* __restrict__ y) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const float4 v = __ldg(x + i);
    y[i] = make_uint2(pack_bf16x2(v.x, v.y), pack_bf16x2(v.z, v.w));
  }
}

__global__ void vae_pad_weight_kernel(const __nv_bfloat16* __restrict__ src, int Cout, int taps, int Cin, int Coutp,
                                      int Cp, __nv_bfloat16* __restrict__ dst) {
  const long long n = static_cast<long long>(Coutp) * taps * Cp;
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const int c = static_cast<int>(i % Cp);
  const int tap = static_cast<int>((i / Cp) % taps);
  const int o = static_cast<int>(i / (static_cast<long long>(Cp) * taps));
  dst[i] = (o < Cout && c < Cin) ? src[(static_cast<long long>(o) * taps + tap) * Cin + c] : __float2bfloat16(0.f);
}

inline unsigned blocks(long long n, int t) { return static_cast<unsigned>((n + t - 1) / t); }
}  // namespace

cudaError_t vae_unpatchify(const float* lat, int F, int Ht, int Wt, const float* mean, const float* stdv,
                           __nv_bfloat16* z, int zc, cudaStream_t stream) {
  const long long nvox = static_cast<long long>(F) * 4 * Ht * Wt;
  if (nvox == 0) return cudaSuccess;
  if (zc != 32 && zc != 64) return cudaErrorInvalidValue;
  vae_unpatchify_kernel<<<blocks(nvox, 256), 256, 0, stream>>>(lat, F, Ht, Wt, mean, stdv, z, zc);
  return cudaGetLastError();
}

cudaError_t vae_rmsnorm_silu(const float* x, const __nv_bfloat16* x_bf16, long long nvox, int C, int Cp,
                             const __nv_bfloat16* gamma, __nv_bfloat16* y, cudaStream_t stream) {
  if (nvox == 0) return cudaSuccess;
  if (Cp % 8 || Cp > 512 || C > Cp) return cudaErrorInvalidValue;
  if (x_bf16)
    vae_rmsnorm_silu_kernel<false><<<blocks(nvox * 32, 256), 256, 0, stream>>>(x_bf16, nvox, C, Cp, gamma, y);
  else
    vae_rmsnorm_silu_kernel<true><<<blocks(nvox * 32, 256), 256, 0, stream>>>(x, nvox, C, Cp, gamma, y);
  return cudaGetLastError();
}

cudaError_t vae_cast_bf16(const float* x, long long n, __nv_bfloat16* y, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  if (n % 4) return cudaErrorInvalidValue;
  const long long n4 = n / 4;
  const long long b = std::min<long long>(blocks(n4, 256), 148LL * 32);
  vae_cast_bf16_kernel<<<static_cast<unsigned>(b), 256, 0, stream>>>(reinterpret_cast<const float4*>(x), n4,
                                                                       reinterpret_cast<uint2*>(y));
  return cudaGetLastError();
}

cudaError_t vae_upsample2(const float* x, const __nv_bfloat16* x_bf16, int T, int H, int W, int Cp,
                          __nv_bfloat16* y, cudaStream_t stream) {
  const long long total = static_cast<long long>(T) * 4 * H * W * (Cp / 8);
  if (total == 0) return cudaSuccess;
  if (Cp % 8) return cudaErrorInvalidValue;
  if (x_bf16)
    vae_upsample2_kernel<false><<<blocks(total, 256), 256, 0, stream>>>(x_bf16, T, H, W, Cp, y);
  else
    vae_upsample2_kernel<true><<<blocks(total, 256), 256, 0, stream>>>(x, T, H, W, Cp, y);
  return cudaGetLastError();
}

cudaError_t vae_pad_weight(const __nv_bfloat16* src, int Cout, int taps, int Cin, int Coutp, int Cp,
                           __nv_bfloat16* dst, cudaStream_t stream) {
  const long long n = static_cast<long long>(Coutp) * taps * Cp;
  vae_pad_weight_kernel<<<blocks(n, 256), 256, 0, stream>>>(src, Cout, taps, Cin, Coutp, Cp, dst);
  return cudaGetLastError();
}

}  // namespace gs
