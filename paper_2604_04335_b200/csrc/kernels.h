// Host-side launchers of the sm_100a kernels (internal to libgs.so; not part of the C-ABI).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

namespace gs {

// ----------------------------------------------------------------- GEMM (gemm.cu)
// C[M,N] = A[M,K] (bf16, row-major, K contiguous) x W[N,K]^T (bf16, row-major) + epilogue.
// Requirements: K % 64 == 0, N % 32 == 0, lda/ldw multiples of 8 elements, 16-B aligned bases.
enum EpiKind : int {
  EPI_BF16 = 0,        // out bf16 [M, ldo] = acc + bias
  EPI_GELU_BF16 = 1,   // out bf16 = GELU_tanh(acc + bias)
  EPI_F32 = 2,         // out fp32 = acc + bias
  EPI_RESID_F32 = 3,   // out fp32 += (gate_a[n] + gate_b[req(m)*gate_b_stride + n]) * (acc + bias)
  EPI_EULER_F32 = 4,   // out fp32 += dsig[req(m)] * (acc + bias)
  EPI_ADD_F32 = 5,     // out fp32 += acc + bias (ungated residual: text cross-attention output)
};

struct EpiParams {
  void* out;
  int ldo;                    // elements
  const __nv_bfloat16* bias;  // [N] or null
  const float* gate_a;        // [N]
  const float* gate_b;        // [B, stride]
  int gate_b_stride;
  const int* row_req;         // [M] request index of each row
  float dsig[8];              // per-request sigma_{i+1} - sigma_i
  int group_m;                // tile rasterisation band (M-tiles); set by the launcher
  // EPI_BF16 only, optional: for output columns < ssq_cols, ssq[row * (ssq_cols / 32) + col / 32]
  // = the sum over that 32-column chunk of (acc + bias)^2 in fp32 (fixed order; chunks are 32-column aligned for
  // every tile width), so the qk-RMSNorm needs no pass of its own over q and k
  float* ssq;
  int ssq_cols;
};

// Programmatic dependent launch for the step's GEMM / attention / row kernels (elementwise.cu):
// on by default; env GS_PDL=0 or gs_set_option "pdl" 0 turns it off (process-wide).
bool pdl_enabled();
extern std::atomic<int> g_pdl;
// Process-wide GEMM pair-tile width override (0 = automatic, 192 or 256; gs_set_option "gemm_bn").
extern std::atomic<int> g_gemm_bn_override;
// Returns cudaError_t; builds the TMA descriptors on the host.
cudaError_t gemm_bf16_tc(int epi, int M, int N, int K, const void* A, int lda, const void* W,
                         int ldw, const EpiParams& ep, int num_sms, cudaStream_t stream);

// ----------------------------------------------------------------- attention (attention.cu)
// O[r, h, :] = softmax(Q_h K_h^T / sqrt(d)) V_h over each request's own rows (block-diagonal).
// Q/K/V/O: bf16 [rows, heads, d] with row strides (elements) *_rs; seq_off/seq_len per request
// (host arrays, nreq <= 64).
// Output scatter (fused head->seq exchange): with nown > 0 the output row of token
// t of segment r (t = row - seq_off[r]) is stored at base[r][i] + t * o_rs + head * d for the
// owner i = max{i < nown : lo[r][i] <= t} (peer memory over NVLink, or a local buffer); O is
// then unused.
constexpr int OSC_MAX_REQ = 16;
struct OScatter {
  int nown;
  int lo[OSC_MAX_REQ][8];
  __nv_bfloat16* base[OSC_MAX_REQ][8];
};
cudaError_t attention_tc(const void* Q, const void* K, const void* V, void* O, int heads, int d,
                         int q_rs, int kv_rs, int o_rs, const int* seq_off, const int* seq_len,
                         int nreq, int num_sms, cudaStream_t stream, const OScatter* scatter = nullptr,
                         int v_rs = 0);  // V's row stride when it differs from K's (0: kv_rs)
// General form: segment r's q_len[r] query rows (from q_off[r]) attend to its kv_len[r] key/value
// rows (from kv_off[r]) -- text cross-attention uses a separate context K/V buffer.
cudaError_t attention_tc_segments(const void* Q, const void* K, const void* V, void* O, int heads, int d,
                                  int q_rs, int kv_rs, int o_rs, const int* q_off, const int* q_len,
                                  const int* kv_off, const int* kv_len, int nreq, cudaStream_t stream,
                                  const OScatter* scatter = nullptr, int v_rs = 0);

// ----------------------------------------------------------------- element-wise (elementwise.cu)
// out[m, :] = LN(x[m, :]) * (1 + sc) + sh, sh = sh_a + sh_b[req(m)*b_stride], same for sc.
cudaError_t ln_modulate(const float* x, int M, int D, const float* sh_a, const float* sh_b,
                        const float* sc_a, const float* sc_b, int b_stride, const int* row_req,
                        float eps, __nv_bfloat16* out, cudaStream_t stream);

// qk-RMSNorm over D, 3-axis RoPE, and pack of q/k/v into the per-destination send layout
// [dest j][row][H_j][d] (dest_off[j] = element offset of chunk j, heads split contiguously).
struct RopeParams {
  const int* row_req;    // [M]
  const int* row_tok;    // [M] request-local token index
  const int* req_grid;   // [B * 3] (F_t, H_t, W_t)
  const float2* cs_tab;  // [P_MAX][d/2] (cos, sin) of pos * freq(slot)
  const int* slot_axis;  // [d/2] axis (0 = f, 1 = h, 2 = w) of each pair slot
  int p_max;
};
constexpr int kMaxChunks = 64;  // p + partial heads (the USP hybrid cuts every head: 8 + 40 at Wan-14B)
struct PackParams {
  int ndest;              // pack chunks: p full-head chunks + one per partial head (<= kMaxChunks)
  int head_off[65];       // head_off[j]..head_off[j+1]: heads of chunk j
  long long dest_off[64]; // element offset of chunk j in each send buffer
  int rows;               // M (local rows; chunk j is [rows][H_j][d])
  // peer-store mode (fused seq->head exchange): chunk j goes straight into the
  // RECV buffers of the position holding it (peer memory over NVLink, or a local buffer), local
  // row m of sequence s (the s with seq_lo[s] <= m: sequences are contiguous row segments; with
  // CFG a request has two) as row m + row_delta[s] of [rows_full][H_j][d]; q_out / k_out / v_out
  // and dest_off are then unused.
  int peer;
  int nseq;
  int seq_lo[16];
  __nv_bfloat16* dst_q[16];
  __nv_bfloat16* dst_k[16];
  __nv_bfloat16* dst_v[16];
  long long row_delta[16];
};
// ssq (optional, D > 2048, qk_uses_ssq): the QKV GEMM's per-32-column sums of squares of q | k ([M][2D / 32] fp32); the row
// sums are then formed from it and q, k are read once.
cudaError_t qk_norm_rope_pack(const __nv_bfloat16* qkv, int M, int D, int heads,
                              const __nv_bfloat16* g_q, const __nv_bfloat16* g_k, float eps,
                              const RopeParams& rp, const PackParams& pk, __nv_bfloat16* q_out,
                              __nv_bfloat16* k_out, __nv_bfloat16* v_out, cudaStream_t stream,
                              const float* ssq = nullptr);
// Whether qk_norm_rope_pack uses the GEMM's sums of squares at this D (the QKV GEMM must then produce them).
bool qk_uses_ssq(int D);

// Time embedding for B requests: e0 = W_t2 SiLU(W_t1 s(t) + b) + b, e = W_tp SiLU(e0) + b.
struct TimeEmbedW {
  const __nv_bfloat16 *w_t1, *b_t1, *w_t2, *b_t2, *w_tp, *b_tp;
  int D, freq_dim;
};
cudaError_t time_embed(const TimeEmbedW& w, int B, const float* t_host /*B*/, float* scratch,
                       float* e0, float* e, cudaStream_t stream);

cudaError_t f32_to_bf16(const float* in, __nv_bfloat16* out, long long n, cudaStream_t stream);

// out[m, :] = in[m, :D] * rsqrt(mean(in[m, :D]^2) + eps) * g  (bf16 in with row stride ld_in,
// bf16 out dense [M, D]); fixed-order reduction as in the other row kernels.
cudaError_t rmsnorm_rows(const __nv_bfloat16* in, int ld_in, int M, int D, const __nv_bfloat16* g, float eps,
                         __nv_bfloat16* out, cudaStream_t stream);
// Classifier-free guidance + Euler on n floats: z += dsig * (vu + g (vc - vu)); vu == null: z += dsig vc.
// z2 (optional) receives the same updated values (the uncond branch's rows of the shared latent).
cudaError_t cfg_euler(float* z, float* z2, const float* vc, const float* vu, long long n, float dsig, float g,
                      cudaStream_t stream);

// ----------------------------------------------------------------- peer barrier (elementwise.cu)
// Cross-GPU step barrier of the fused exchanges: thread t stores val[t] into slot[t] (a flag word
// in a peer's memory) with system-scope release after a system fence (signal), or spins with
// system-scope acquire until *slot[t] >= val[t] (wait; traps after ~20 s instead of hanging).
struct PeerFlags {
  int n;
  unsigned long long* slot[8];
  unsigned long long val[8];
};
cudaError_t peer_signal(const PeerFlags& f, cudaStream_t stream);
cudaError_t peer_wait(const PeerFlags& f, cudaStream_t stream);
// Probe variant of peer_wait: gives up after ~timeout_ms and stores 1 (all flags arrived) or 0 to
// *ok (device int) instead of trapping -- used once per gs_run_steps to prove the IPC mappings
// before any data-path kernel stores into peer memory.
cudaError_t peer_wait_probe(const PeerFlags& f, int timeout_ms, int* ok, cudaStream_t stream);

// ----------------------------------------------------------------- VAE decode (conv.cu, vae_kernels.cu)
// Implicit-GEMM causal 3-D convolution (oracle/vae.py causal_conv3d): x bf16 [T][H][W][Cp]
// channels-last, w bf16 [Coutp][kt][kh][kw][Cp], bias bf16 [Coutp], optional residual bf16 or fp32
// [T][H][W][Coutp] added in fp32.  Cp, Coutp multiples of 32.  Output modes:
enum ConvOut : int {
  CONV_OUT_BF16 = 0,             // out bf16 [T][H][W][out_cs], channels [0, Coutp)
  CONV_OUT_TIME_INTERLEAVE = 1,  // temporal upsample: channels [0, out_real) -> frame 2t+1,
                                 // [out_real, 2 out_real) -> frame 2t+2 (out bf16 [.][H][W][out_cs])
  CONV_OUT_F32_CLAMP = 2,        // out fp32 [T][H][W][out_real] = clamp(acc + b, -1, 1), channels < out_real
  CONV_OUT_F32 = 3,              // out fp32 [T][H][W][out_cs] (the decoder's fp32 residual stream)
  CONV_OUT_NONE = 4,             // no main output (only the fused norm output below)
};
struct ConvParams {
  int T, H, W, Cp, kt, kh, kw, Coutp;
  const __nv_bfloat16* bias;
  const void* resid;   // bf16 or (resid_f32) fp32 [T][H][W][Coutp], or null
  void* out;
  int out_cs, mode, out_real;
  int resid_f32;
  // Fused RMS norm + SiLU of the result (the next residual block's norm, oracle/vae.py rms_norm_c +
  // silu): with norm_gamma set, y = SiLU(v sqrt(norm_c) / max(||v||, 1e-12) gamma) over the first norm_c
  // channels of v = acc + b (+ resid) is also written, bf16 [T][H][W][Coutp] to norm_out (pad channels
  // 0).  Needs one N tile per voxel (conv_bn(Coutp) == Coutp) and mode F32 or NONE (NONE: no resid).
  const __nv_bfloat16* norm_gamma;
  __nv_bfloat16* norm_out;
  int norm_c;
};
// N tile width of conv3d_tc for Coutp output channels (a fused norm needs conv_bn(Coutp) == Coutp).
int conv_bn(int Coutp);
cudaError_t conv3d_tc(const void* x, const void* w, const ConvParams& cp, int num_sms, cudaStream_t stream);
// DiT latent [F*Ht*Wt, 64] fp32 (features (c, pt, ph, pw)) -> z bf16 [F][2Ht][2Wt][zc] (zc = 32 or 64):
// z = lat * std[c] + mean[c] for the 16 channels, channels 16..zc-1 = 0 (reading V6).
cudaError_t vae_unpatchify(const float* lat, int F, int Ht, int Wt, const float* mean, const float* stdv,
                           __nv_bfloat16* z, int zc, cudaStream_t stream);
// y = SiLU(x sqrt(C) / max(||x||, 1e-12) gamma) per voxel over the C real channels of Cp (pad -> 0);
// x fp32 (the residual stream) or bf16 (x_bf16 != null).
cudaError_t vae_rmsnorm_silu(const float* x, const __nv_bfloat16* x_bf16, long long nvox, int C, int Cp,
                             const __nv_bfloat16* gamma, __nv_bfloat16* y, cudaStream_t stream);
// Nearest x2 in H and W: y bf16 [T][2H][2W][Cp] from x fp32 (RNE) or x_bf16 [T][H][W][Cp].
cudaError_t vae_upsample2(const float* x, const __nv_bfloat16* x_bf16, int T, int H, int W, int Cp,
                          __nv_bfloat16* y, cudaStream_t stream);
// y bf16 = RNE(x fp32), n elements (n % 4 == 0).
cudaError_t vae_cast_bf16(const float* x, long long n, __nv_bfloat16* y, cudaStream_t stream);
// Dense [Cout][taps][Cin] bf16 -> padded [Coutp][taps][Cp] (zeros elsewhere).
cudaError_t vae_pad_weight(const __nv_bfloat16* src, int Cout, int taps, int Cin, int Coutp, int Cp,
                           __nv_bfloat16* dst, cudaStream_t stream);

// ----------------------------------------------------------------- RNG (rng.cu)
// Counter RNG of DESIGN.md "Input recipe" (independent re-implementation of synth/rng.py).
enum RngKind : int { RNG_BF16_SCALED = 0, RNG_BF16_GAIN = 1, RNG_F32_SCALED = 2 };
cudaError_t rng_fill(void* out, long long n, uint64_t seed, uint32_t tensor_id, int kind,
                     float scale, cudaStream_t stream);
// Standard-normal (Irwin-Hall(4)) values rounded to bf16: synthetic prompt embeddings.
cudaError_t rng_normal_bf16(__nv_bfloat16* out, long long n, uint64_t seed, uint32_t tensor_id,
                            cudaStream_t stream);
// z[i, c] for tokens [tok_lo, tok_lo + ntok) of a request's [n, 64] noise latent.
cudaError_t rng_noise(float* out, long long tok_lo, long long ntok, int channels, uint64_t seed,
                      cudaStream_t stream);

}  // namespace gs
