// tcgen05 implicit-GEMM causal 3-D convolution for the VAE decode stage (
// oracle: oracle/vae.py causal_conv3d, reading V2):
//   y[t, h, w, co] = b[co] + sum_{dt, dh, dw, ci} W[co, dt, dh, dw, ci] x[t + dt - (kt-1), h + dh - ph, w + dw - pw, ci]
// with zero padding (kt - 1 frames before the sequence; ph = (kh-1)/2, pw = (kw-1)/2 on both sides).
//
// Design (B200-first; the GEMM of gemm.cu with a convolutional A operand):
//   * activations channels-last bf16 [T][H][W][Cp] (Cp = channels padded to a multiple of 64);
//     weights bf16 [Coutp][kt][kh][kw][Cp], i.e. the K index of the implicit GEMM is tap-major,
//     channel-minor (K = kt kh kw Cp);
//   * M tile of a CTA = 128 output voxels = a 4 (h) x 32 (w) patch of one frame; a CTA pair
//     (cta_group::2, M = 256 MMAs) takes 8 x 32; one 4-D TMA box {64 ch, 32 w, 4 h, 1 t} per K block
//     and tap loads the patch shifted by the tap with the conv's zero padding done by TMA's
//     out-of-bounds fill (negative / past-the-end coordinates read zeros), already in the 128B-
//     swizzled K-major layout the UMMA descriptor expects (128 rows x 128 B);
//   * persistent CTA pairs, warp 0 TMA producer, warp 1 TMEM owner + MMA issuer (leader), warps 2-5
//     epilogue from two TMEM accumulators (epilogue of tile i overlaps the MMAs of tile i + 1);
//   * epilogue per output voxel (TMEM lane = voxel): + bias, + residual (bf16 or fp32, optional), then
//     one of: bf16 store (64 B per thread per 32-channel chunk); fp32 store (the decoder's residual
//     stream, 128 B per chunk); the temporal-upsample interleave (the
//     two channel halves of frame t go to output frames 2t + 1, 2t + 2; reading V5); fp32 clamp to
//     [-1, 1] of the first `out_real` channels (the decoder output, reading V7); optionally also the
//     next residual block's RMS norm + SiLU of the same values (ConvParams::norm_*: a second pass over
//     the voxel's channels once their square sum is known -- one TMEM lane holds all of a voxel's
//     channels when one N tile spans Coutp), which removes the decoder's stand-alone norm passes.
// Each output depends only on its own inputs; no split-K, no atomics.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>

#include "kernels.h"
#include "ptx.cuh"
#include "tma.h"

namespace gs {

namespace {
constexpr int CBM = 128;                 // voxels per CTA (pair: 256)
constexpr int PATCH_W = 32, PATCH_H = 4;  // CTA patch (pair: 8 rows)
constexpr int CTHREADS = 192;

// KB = channels per TMA box / swizzle atom row: 64 (rows of 128 B, 128-byte swizzle) or 32 (rows of
// 64 B, 64-byte swizzle) for channel counts = 32 mod 64 (the 96-channel last stage runs unpadded).
// NS boxes per pipeline stage (a 96-channel tap = 3 x 32 in one stage, so each barrier round trip
// still feeds 6 MMAs).
// WR (W-row reuse, kw = 3 convolutions): the CTA's 128 voxels are one h-row of 128 w, and one TMA box
// of 130 w (the row plus its +-1 halo) per (dt, dh, channel block) serves all three dw taps -- the
// UMMA descriptor of tap dw starts dw rows into the box (uniform 8-row core groups; UMMA applies the
// swizzle to absolute shared-memory address bits like TMA, so a row-shifted start with the matrix
// base-offset field left 0 reads what TMA wrote -- measured: the field set to the start's 128-byte
// line gives wrong results).
// A-operand traffic per tile drops from kt kh kw to kt kh boxes.
template <int BN, int KB, int NS, bool WR = false>
struct CCfg {
  static constexpr int A_ROWS = WR ? CBM + 2 : CBM;                          // rows TMA writes per box
  static constexpr int A_SUB = (A_ROWS * KB * 2 + 1023) / 1024 * 1024;       // swizzle-atom aligned
  static constexpr int TAPS = WR ? 3 : 1;                                    // dw taps per stage
  static constexpr int B_SUB = (BN / 2) * KB * 2;
  static constexpr int A_BYTES = NS * A_SUB;
  static constexpr int B_BYTES = TAPS * NS * B_SUB;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGE_TX = NS * A_ROWS * KB * 2 + B_BYTES;            // bytes TMA delivers
  static constexpr int MAXST = 8;
  static constexpr int STAGES = (200 * 1024) / STAGE_BYTES > MAXST ? MAXST : (200 * 1024) / STAGE_BYTES;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 1024;
  static constexpr uint32_t TMEM_COLS = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128
                                      : 2 * BN <= 256 ? 256 : 512;
  static_assert(SMEM_BYTES <= 232448, "shared memory");
  static_assert(A_SUB % 1024 == 0 && B_SUB % 512 == 0 && STAGE_BYTES % 1024 == 0, "swizzle atom alignment");
};

// Shared-memory descriptor of a K-major operand with KB-channel rows (128B or 64B swizzle).
template <int KB>
__device__ __forceinline__ uint64_t sdesc_kb(uint32_t saddr) {
  if (KB == 64) return sdesc_sw128(saddr, 16, 1024);
  uint64_t d = 0;  // 64-byte swizzle (layout type 4): 8-row core groups of 512 B
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1) << 16;
  d |= static_cast<uint64_t>(512 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(4) << 61;
  return d;
}

__device__ __forceinline__ void tma_load_4d_2sm(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1,
                                                int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

struct TileGeom {
  int num_hb, num_wb, num_m, num_n;  // h blocks of 2 * patch_h rows (pair), w blocks of patch_w
  __device__ void coords(int tile, int& t, int& hb, int& wb, int& nb) const {
    // n fastest (the A patch is reused from L2 by the pair's consecutive N tiles)
    nb = tile % num_n;
    const int m = tile / num_n;
    wb = m % num_wb;
    hb = (m / num_wb) % num_hb;
    t = m / (num_wb * num_hb);
  }
};

template <int BN, int KB, int NS, bool WR>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(CTHREADS, 1)
    conv3d_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ ConvParams cp) {
  using C = CCfg<BN, KB, NS, WR>;
  constexpr int PH = WR ? 1 : PATCH_H, PW = WR ? CBM : PATCH_W;  // CTA patch (rows x cols)
  constexpr int CA_BYTES = C::A_BYTES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* full = bars;                     // [STAGES] leader's count both CTAs' bytes
  uint64_t* empty = bars + C::STAGES;        // [STAGES] per CTA (multicast commit)
  uint64_t* tfull = bars + 2 * C::STAGES;    // [2]
  uint64_t* tempty = bars + 2 * C::STAGES + 2;  // [2] leader's: 4 epilogue warps x 2 CTAs
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * C::STAGES + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  TileGeom g;
  g.num_hb = (cp.H + 2 * PH - 1) / (2 * PH);
  g.num_wb = (cp.W + PW - 1) / PW;
  g.num_m = cp.T * g.num_hb * g.num_wb;
  g.num_n = cp.Coutp / BN;
  const int num_tiles = g.num_m * g.num_n;
  const int cpb = cp.Cp / (KB * NS);  // channel stage-blocks per tap
  const int num_k = cp.kt * cp.kh * (WR ? 1 : cp.kw) * cpb;  // pipeline stages per tile

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
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
  if (warp == 1) tmem_alloc_2sm(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();
  pdl_launch_dependents();

  if (warp == 0) {
    if (lane == 0) {  // producer (both CTAs): this CTA's voxel patch per tap and its weight half
      int stage = 0;
      uint32_t phase = 0;
      const int ph = (cp.kh - 1) / 2, pw = (cp.kw - 1) / 2;
      for (int tile = pair; tile < num_tiles; tile += npairs) {
        int t, hb, wb, nb;
        g.coords(tile, t, hb, wb, nb);
        const int h0 = hb * 2 * PH + static_cast<int>(rank) * PH, w0 = wb * PW;
        int cb = 0, dw = 0, dh = 0, dt = 0;
        for (int kb = 0; kb < num_k; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * C::STAGE_BYTES;
          mbar_arrive_expect_tx_cluster(mapa_shared(smem_u32(&full[stage]), 0), C::STAGE_TX);
#pragma unroll
          for (int sub = 0; sub < NS; ++sub) {
            const int ch = (cb * NS + sub) * KB;
            // WR: the row with its halo, [w0 - pw, w0 - pw + 130), once for all dw taps
            tma_load_4d_2sm(&tmA, &full[stage], sa + sub * C::A_SUB, ch, w0 + (WR ? 0 : dw) - pw, h0 + dh - ph,
                            t + dt - (cp.kt - 1));
#pragma unroll
            for (int q = 0; q < C::TAPS; ++q) {  // weights of tap (dt, dh, dw + q), K = tap * Cp + ch
              const int tap = (dt * cp.kh + dh) * cp.kw + dw + q;
              tma_load_2d_2sm(&tmB, &full[stage], sa + CA_BYTES + (q * NS + sub) * C::B_SUB, tap * cp.Cp + ch,
                              nb * BN + static_cast<int>(rank) * (BN / 2));
            }
          }
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
          if (++cb == cpb) {  // K order: tap-major (dt, dh, dw), channel block minor
            cb = 0;
            if (WR || ++dw == cp.kw) {
              dw = 0;
              if (++dh == cp.kh) { dh = 0; ++dt; }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {  // MMA issuer (leader CTA)
      constexpr uint32_t idesc = idesc_bf16(2 * CBM, BN, 0, 0);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = pair; tile < num_tiles; tile += npairs, ++it) {
        const int as = it & 1;
        mbar_wait(&tempty[as], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + as * BN;
        for (int kb = 0; kb < num_k; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * C::STAGE_BYTES);
          const uint32_t sb = sa + CA_BYTES;
#pragma unroll
          for (int q = 0; q < C::TAPS * NS * (KB / 16); ++q) {
            const int tq = q / (NS * (KB / 16)), sub = (q / (KB / 16)) % NS, kk = q % (KB / 16);
            const uint32_t a = sa + sub * C::A_SUB + tq * (KB * 2) + kk * 32;  // WR: dw = tq rows down
            mma_ss_2sm(d_tmem, sdesc_kb<KB>(a),
                       sdesc_kb<KB>(sb + (tq * NS + sub) * C::B_SUB + kk * 32), idesc, (kb | q) != 0);
          }
          mma_commit_2sm_mc(&empty[stage], 0x3);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit_2sm_mc(&tfull[as], 0x3);
      }
    }
  } else {
    // epilogue: warp (2..5) % 4 = TMEM lane quarter = patch row; lane = patch column
    const int quarter = warp & 3;
    const uint32_t tempty_leader = mapa_shared(smem_u32(&tempty[0]), 0);
    int it = 0;
    for (int tile = pair; tile < num_tiles; tile += npairs, ++it) {
      int t, hb, wb, nb;
      g.coords(tile, t, hb, wb, nb);
      const int as = it & 1;
      mbar_wait(&tfull[as], (it >> 1) & 1);
      tc_fence_after();
      // TMEM lane (quarter * 32 + lane) = voxel of the CTA patch, row-major over PH x PW
      const int pv = quarter * 32 + lane;
      const int h = hb * 2 * PH + static_cast<int>(rank) * PH + pv / PW, w = wb * PW + pv % PW;
      const bool valid = h < cp.H && w < cp.W;
      const long long vox = (static_cast<long long>(t) * cp.H + h) * cp.W + w;
      const uint32_t tbase = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + as * BN;
      // fused norm (host-checked: one N tile per voxel): pass 1 below accumulates the square sum, pass 2
      // writes the normalised activation; with no main output pass 2 re-reads TMEM, so the accumulator
      // is handed back to the MMA issuer only after it
      const bool fuse = cp.norm_gamma != nullptr;
      const bool reread = fuse && cp.mode == CONV_OUT_NONE;
      float ss = 0.f;
      auto add_bias = [&](const uint32_t(&r)[32], int ch0, float(&v)[32]) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          const uint4 braw = __ldg(reinterpret_cast<const uint4*>(cp.bias + ch0 + i));
          const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&braw);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float2 bf = __bfloat1622float2(b2[j]);
            v[i + 2 * j] = __uint_as_float(r[i + 2 * j]) + bf.x;
            v[i + 2 * j + 1] = __uint_as_float(r[i + 2 * j + 1]) + bf.y;
          }
        }
      };
      auto hand_back = [&]() {  // accumulator fully in registers: hand it back to the MMA issuer
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tempty_leader + as * 8);
      };
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        GS_TMEM_LD32(tbase + c * 32, r);
        tmem_ld_wait();
        if (c + 1 == BN / 32 && !reread) hand_back();
        if (!valid) continue;
        const int ch0 = nb * BN + c * 32;
        float v[32];
        add_bias(r, ch0, v);
        if (cp.resid != nullptr && cp.resid_f32) {
          const float4* rp = reinterpret_cast<const float4*>(static_cast<const float*>(cp.resid) + vox * cp.Coutp + ch0);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 r = __ldg(rp + q);
            v[4 * q] += r.x;
            v[4 * q + 1] += r.y;
            v[4 * q + 2] += r.z;
            v[4 * q + 3] += r.w;
          }
        } else if (cp.resid != nullptr) {
          const uint4* rp =
              reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(cp.resid) + vox * cp.Coutp + ch0);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint4 raw = __ldg(rp + q);
            const __nv_bfloat162* r2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float2 rf = __bfloat1622float2(r2[j]);
              v[8 * q + 2 * j] += rf.x;
              v[8 * q + 2 * j + 1] += rf.y;
            }
          }
        }
        if (fuse) {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (ch0 + i < cp.norm_c) ss = fmaf(v[i], v[i], ss);
        }
        if (cp.mode == CONV_OUT_NONE) continue;
        if (cp.mode == CONV_OUT_F32_CLAMP) {
          float* o = static_cast<float*>(cp.out) + vox * cp.out_real;
          for (int i = 0; i < 32 && ch0 + i < cp.out_real; ++i) o[ch0 + i] = fminf(fmaxf(v[i], -1.0f), 1.0f);
          continue;
        }
        if (cp.mode == CONV_OUT_F32) {
          float4* o = reinterpret_cast<float4*>(static_cast<float*>(cp.out) + vox * cp.out_cs + ch0);
#pragma unroll
          for (int q = 0; q < 8; ++q) o[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
          continue;
        }
        long long dst_vox = vox;
        int dch = ch0;
        if (cp.mode == CONV_OUT_TIME_INTERLEAVE) {  // output frames 2t + 1 (first half), 2t + 2 (second)
          const int half = ch0 >= cp.out_real;
          dch = ch0 - half * cp.out_real;
          dst_vox = (static_cast<long long>(2 * t + 1 + half) * cp.H + h) * cp.W + w;
        }
        uint4* o = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(cp.out) + dst_vox * cp.out_cs + dch);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          o[q] = make_uint4(pack_bf16x2(v[8 * q], v[8 * q + 1]), pack_bf16x2(v[8 * q + 2], v[8 * q + 3]),
                            pack_bf16x2(v[8 * q + 4], v[8 * q + 5]), pack_bf16x2(v[8 * q + 6], v[8 * q + 7]));
      }
      if (fuse) {  // pass 2: y = SiLU(v sqrt(C) / max(||v||, 1e-12) gamma), the same v as pass 1
        const float scale = sqrtf(static_cast<float>(cp.norm_c)) / fmaxf(sqrtf(ss), 1e-12f);
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          const int ch0 = nb * BN + c * 32;
          float v[32];
          if (reread) {
            uint32_t r[32];
            GS_TMEM_LD32(tbase + c * 32, r);
            tmem_ld_wait();
            if (c + 1 == BN / 32) hand_back();
            if (!valid) continue;
            add_bias(r, ch0, v);
          } else {  // F32: v as stored by pass 1 (this thread's own writes; exact)
            if (!valid) continue;
            const float4* src = reinterpret_cast<const float4*>(static_cast<const float*>(cp.out) + vox * cp.out_cs + ch0);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float4 t4 = src[q];
              v[4 * q] = t4.x;
              v[4 * q + 1] = t4.y;
              v[4 * q + 2] = t4.z;
              v[4 * q + 3] = t4.w;
            }
          }
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 32; i += 8) {
            const uint4 graw = __ldg(reinterpret_cast<const uint4*>(cp.norm_gamma + ch0 + i));
            const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&graw);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float2 gf = __bfloat1622float2(g2[j]);
              float u[2];
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int ci = i + 2 * j + e;
                const float n = v[ci] * scale * (e ? gf.y : gf.x);
                u[e] = ch0 + ci < cp.norm_c ? n / (1.0f + __expf(-n)) : 0.f;
              }
              pk[(i + 2 * j) / 2] = pack_bf16x2(u[0], u[1]);
            }
          }
          uint4* o = reinterpret_cast<uint4*>(cp.norm_out + vox * cp.Coutp + ch0);
#pragma unroll
          for (int q = 0; q < 4; ++q) o[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_2sm(tmem_base, C::TMEM_COLS);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 tma_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  return enc;
}

bool make_tma_4d_act(CUtensorMap* m, const void* base, int Cp, int W, int H, int T, int kb, int box_w, int box_h) {
  auto enc = tma_encoder();
  if (!enc) return false;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(Cp), static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(H),
                        static_cast<cuuint64_t>(T)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(Cp) * 2, static_cast<cuuint64_t>(W) * Cp * 2,
                           static_cast<cuuint64_t>(H) * W * Cp * 2};
  cuuint32_t box[4] = {static_cast<cuuint32_t>(kb), static_cast<cuuint32_t>(box_w), static_cast<cuuint32_t>(box_h), 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, kb == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Weights [Coutp][K] bf16 with box {kb, rows}; 128B swizzle for kb = 64, 64B for kb = 32.
bool make_tma_w(CUtensorMap* m, const void* base, long long K, int Coutp, int kb, int rows) {
  if (kb == 64) return make_tma_2d_bf16(m, base, K, Coutp, K * 2, 64, rows);
  auto enc = tma_encoder();
  if (!enc) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(Coutp)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(K) * 2};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(kb), static_cast<cuuint32_t>(rows)};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN, int KB, int NS, bool WR>
cudaError_t launch_conv(const void* x, const void* w, const ConvParams& cp, int num_sms, cudaStream_t stream) {
  using C = CCfg<BN, KB, NS, WR>;
  constexpr int PH = WR ? 1 : PATCH_H, PW = WR ? CBM : PATCH_W;
  CUtensorMap ta, tb;
  if (!make_tma_4d_act(&ta, x, cp.Cp, cp.W, cp.H, cp.T, KB, WR ? C::A_ROWS : PATCH_W, PH))
    return cudaErrorInvalidValue;
  const long long K = static_cast<long long>(cp.kt) * cp.kh * cp.kw * cp.Cp;
  if (!make_tma_w(&tb, w, K, cp.Coutp, KB, BN / 2)) return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(conv3d_tc_kernel<BN, KB, NS, WR>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const long long tiles =
      static_cast<long long>(cp.T) * ((cp.H + 2 * PH - 1) / (2 * PH)) * ((cp.W + PW - 1) / PW) * (cp.Coutp / BN);
  const int pairs = static_cast<int>(std::min<long long>(tiles, num_sms / 2));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(CTHREADS);
  cfg.dynamicSmemBytes = C::SMEM_BYTES;
  cfg.stream = stream;
  cudaLaunchAttribute at;
  at.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at.val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = &at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, conv3d_tc_kernel<BN, KB, NS, WR>, ta, tb, cp);
}
}  // namespace

int conv_bn(int Coutp) {
  if (Coutp % 256 == 0) return 256;
  if (Coutp % 192 == 0) return 192;
  if (Coutp % 128 == 0) return 128;
  if (Coutp % 96 == 0) return 96;
  if (Coutp % 64 == 0) return 64;
  return 32;
}

template <int KB, int NS, bool WR>
cudaError_t launch_bn(const void* x, const void* w, const ConvParams& cp, int num_sms, cudaStream_t stream) {
  switch (conv_bn(cp.Coutp)) {
    case 256: return launch_conv<256, KB, NS, WR>(x, w, cp, num_sms, stream);
    case 192: return launch_conv<192, KB, NS, WR>(x, w, cp, num_sms, stream);
    case 128: return launch_conv<128, KB, NS, WR>(x, w, cp, num_sms, stream);
    case 96: return launch_conv<96, KB, NS, WR>(x, w, cp, num_sms, stream);
    case 64: return launch_conv<64, KB, NS, WR>(x, w, cp, num_sms, stream);
    default: return launch_conv<32, KB, NS, WR>(x, w, cp, num_sms, stream);
  }
}
template <int KB, int NS>
cudaError_t launch_kb(const void* x, const void* w, const ConvParams& cp, int num_sms, cudaStream_t stream) {
  // 3-wide w taps: one halo row box serves all three (WR); other widths tap by tap
  return cp.kw == 3 ? launch_bn<KB, NS, true>(x, w, cp, num_sms, stream)
                    : launch_bn<KB, NS, false>(x, w, cp, num_sms, stream);
}

cudaError_t conv3d_tc(const void* x, const void* w, const ConvParams& cp, int num_sms, cudaStream_t stream) {
  if (cp.T <= 0 || cp.H <= 0 || cp.W <= 0) return cudaSuccess;
  if (cp.Cp % 32 || cp.Coutp % 32 || cp.kt < 1 || cp.kh < 1 || cp.kw < 1 || !cp.bias ||
      (!cp.out && cp.mode != CONV_OUT_NONE))
    return cudaErrorInvalidValue;
  if ((cp.mode == CONV_OUT_BF16 || cp.mode == CONV_OUT_F32) && (cp.out_cs % 8 || cp.out_cs < cp.Coutp))
    return cudaErrorInvalidValue;
  if (cp.mode == CONV_OUT_TIME_INTERLEAVE && (cp.out_real % 32 || 2 * cp.out_real > cp.Coutp || cp.out_cs % 8))
    return cudaErrorInvalidValue;
  if (cp.norm_gamma && (!cp.norm_out || conv_bn(cp.Coutp) != cp.Coutp || cp.norm_c < 1 || cp.norm_c > cp.Coutp ||
                        !(cp.mode == CONV_OUT_F32 || (cp.mode == CONV_OUT_NONE && !cp.resid))))
    return cudaErrorInvalidValue;
  if (cp.mode == CONV_OUT_NONE && !cp.norm_gamma) return cudaErrorInvalidValue;
  // 64-channel K blocks (128B swizzle) when the input channels allow, else 32 (64B swizzle)
  if (cp.Cp % 64 == 0) return launch_kb<64, 1>(x, w, cp, num_sms, stream);
  if (cp.Cp % 96 == 0) return launch_kb<32, 3>(x, w, cp, num_sms, stream);  // 96-channel taps in one stage
  return launch_kb<32, 1>(x, w, cp, num_sms, stream);

}

}  // namespace gs
