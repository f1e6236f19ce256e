// VAE decode stage: host runtime and C-ABI of the decoder.
//
// "GenServe efficiently decouples the two stages, letting the VAE stage always execute on a single
// GPU, while the DiT stage is parallelized via Sequence Parallelism" (§4.3).  The decoder
// is the Wan2.1-VAE-shaped causal 3-D conv decoder of DESIGN.md §NEXT-4 (readings V1-V8), rebuilt
// here from its definition (the same module walk as synth/vae.py, written independently):
//   unpatchify + de-normalise -> post 1x1x1 -> conv_in 3x3x3 -> mid residual blocks ->
//   per stage {residual blocks, [temporal x2 time-conv], [nearest x2 + 1x3x3 conv]} ->
//   RMS norm + SiLU -> conv_out 3x3x3 -> clamp.
// Every convolution is conv3d_tc (tcgen05 implicit GEMM, conv.cu); norms, upsampling and the
// unpatchify are the HBM-bound kernels of vae_kernels.cu.  Activations bf16 channels-last with
// channels padded to multiples of 32 (pad channels are zero; padded weight rows / columns are zero).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "runtime.h"

using namespace gs;

namespace {

int vfail(gs_ctx* c, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (tl_err) {
    *tl_err = buf;
  } else if (c) {
    std::lock_guard<std::mutex> g(c->err_mu);
    c->err = buf;
  }
  return code;
}

#define VCK(call)                                                                                   \
  do {                                                                                              \
    cudaError_t e_ = (call);                                                                        \
    if (e_ != cudaSuccess) return vfail(c, GS_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call,    \
                                        cudaGetErrorString(e_));                                    \
  } while (0)
#define VRET(call)                \
  do {                            \
    int rc_ = (call);             \
    if (rc_ != GS_OK) return rc_; \
  } while (0)

// channels padded to a multiple of 32 (the conv's K blocks are 64 or 32 channels wide)
inline int padc(int c) { return (c + 31) / 32 * 32; }

int vlocal(gs_ctx* c, int rank) {
  if (c->emulated) return (rank >= 0 && rank < c->world) ? rank : -1;
  return rank == c->my_rank ? 0 : -1;
}

// ------------------------------------------------------------------ weights
struct Gen {
  gs_ctx* c;
  Vae* v;
  cudaStream_t s;
  int module = 0;  // walk index: tensor id 200 + 4 * module + slot
  int alloc(void** p, size_t bytes) {
    if (cudaMalloc(p, bytes) != cudaSuccess) {
      cudaGetLastError();
      return vfail(c, GS_ENOMEM, "VAE weight alloc (%zu B) failed", bytes);
    }
    v->allocs.push_back(*p);
    return GS_OK;
  }
  int conv(VaeConv& cv, int cin, int cout, int kt, int kh, int kw) {
    cv.cin = cin;
    cv.cout = cout;
    cv.kt = kt;
    cv.kh = kh;
    cv.kw = kw;
    cv.cp = padc(cin);
    cv.coutp = padc(cout);
    const int taps = kt * kh * kw;
    const long long dense = static_cast<long long>(cout) * taps * cin;
    const uint32_t tid = 200 + 4 * module++;
    void* tmp = nullptr;
    if (cudaMalloc(&tmp, dense * 2) != cudaSuccess) {
      cudaGetLastError();
      return vfail(c, GS_ENOMEM, "VAE weight staging failed");
    }
    int rc = GS_OK;
    void *w = nullptr, *b = nullptr;
    if ((rc = alloc(&w, static_cast<size_t>(cv.coutp) * taps * cv.cp * 2)) == GS_OK &&
        (rc = alloc(&b, static_cast<size_t>(cv.coutp) * 2)) == GS_OK) {
      const float scale = static_cast<float>(std::sqrt(3.0 / (static_cast<double>(cin) * taps)));
      cudaError_t e = rng_fill(tmp, dense, v->desc.weight_seed, tid, RNG_BF16_SCALED, scale, s);
      if (e == cudaSuccess)
        e = vae_pad_weight(static_cast<bf16*>(tmp), cout, taps, cin, cv.coutp, cv.cp, static_cast<bf16*>(w), s);
      if (e == cudaSuccess) e = cudaMemsetAsync(b, 0, static_cast<size_t>(cv.coutp) * 2, s);
      if (e == cudaSuccess) e = rng_fill(b, cout, v->desc.weight_seed, tid + 1, RNG_BF16_SCALED, 0.1f, s);
      if (e == cudaSuccess) e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) rc = vfail(c, GS_ECUDA, "VAE weights: %s", cudaGetErrorString(e));
    }
    cudaFree(tmp);
    cv.w = static_cast<bf16*>(w);
    cv.b = static_cast<bf16*>(b);
    return rc;
  }
  int norm(VaeNorm& n, int ch) {
    n.c = ch;
    void* g = nullptr;
    VRET(alloc(&g, static_cast<size_t>(ch) * 2));
    cudaError_t e = rng_fill(g, ch, v->desc.weight_seed, 200 + 4 * module++, RNG_BF16_GAIN, 0.f, s);
    if (e != cudaSuccess) return vfail(c, GS_ECUDA, "VAE gamma: %s", cudaGetErrorString(e));
    n.gamma = static_cast<bf16*>(g);
    return GS_OK;
  }
  int res(VaeRes& r, int cin, int cout) {
    VRET(norm(r.n1, cin));
    VRET(conv(r.c1, cin, cout, 3, 3, 3));
    VRET(norm(r.n2, cout));
    VRET(conv(r.c2, cout, cout, 3, 3, 3));
    if (cin != cout) VRET(conv(r.skip, cin, cout, 1, 1, 1));
    return GS_OK;
  }
};

// ------------------------------------------------------------------ decode
struct Act {  // a channels-last activation view
  bf16* p;
  int T, H, W, C, Cp;
  long long vox() const { return static_cast<long long>(T) * H * W; }
};

struct Decoder {
  gs_ctx* c;
  Vae* v;
  cudaStream_t s;
  bool dry;                 // sizing pass: record the largest use of each buffer role, launch nothing
  size_t need[4] = {0, 0, 0, 0};
  // roles: 0 X (fp32 residual stream), 1 N (bf16: norm output / bf16 copy / upsample), 2 H (bf16: conv1
  // output, latent, time-conv output), 3 S (fp32 skip-path residual)
  void* buf[4] = {nullptr, nullptr, nullptr, nullptr};
  static size_t esize(int r) { return r == 0 || r == 3 ? 4 : 2; }

  template <class T>
  T* role(int r, size_t elems) {
    need[r] = std::max(need[r], elems);
    return static_cast<T*>(buf[r]);
  }
  int ck(cudaError_t e, const char* what) {
    return e == cudaSuccess ? GS_OK : vfail(c, GS_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  }
  // Buffer role holding SiLU(norm(X)) for the next consumer (fused into the producing conv's
  // epilogue), or -1.  Roles 1 and 2 alternate so a conv never writes the buffer it reads.
  int ready = -1;
  static bool fusable(int coutp) { return conv_bn(coutp) == coutp; }
  // one convolution; x bf16 [T][H][W][x_cp]; with `nrm` its epilogue also writes SiLU(nrm(v)) to nout
  int conv(const VaeConv& cv, const bf16* x, int T, int H, int W, int x_cp, void* out, int mode,
           const void* resid = nullptr, bool resid_f32 = false, int out_real = 0, int out_cs = 0,
           const VaeNorm* nrm = nullptr, bf16* nout = nullptr) {
    if (dry) return GS_OK;
    ConvParams p{};
    p.T = T;
    p.H = H;
    p.W = W;
    p.Cp = x_cp;
    p.kt = cv.kt;
    p.kh = cv.kh;
    p.kw = cv.kw;
    p.Coutp = cv.coutp;
    p.bias = cv.b;
    p.resid = resid;
    p.resid_f32 = resid_f32 ? 1 : 0;
    p.out = out;
    p.out_cs = out_cs ? out_cs : cv.coutp;
    p.mode = mode;
    p.out_real = out_real;
    if (nrm) {
      p.norm_gamma = nrm->gamma;
      p.norm_out = nout;
      p.norm_c = nrm->c;
    }
    return ck(conv3d_tc(x, cv.w, p, c->num_sms, s), "conv3d");
  }
  // residual block on the fp32 stream X [T][H][W][cp] (C real channels); returns the new width.  `next`
  // is the norm applied to the block's output by the following consumer (the next block's norm1 or
  // norm_out), fused into conv2's epilogue when the width allows; null when X is read raw next.
  int res(const VaeRes& r, int T, int H, int W, int& C, int& cp, const VaeNorm* next) {
    const size_t vox = static_cast<size_t>(T) * H * W;
    const size_t wide = vox * std::max(cp, r.c1.coutp);
    float* X = role<float>(0, wide);
    const void* resid = X;
    if (r.skip.cout) {  // shortcut conv of x (bf16 copy of the stream) -> S (fp32)
      float* S = role<float>(3, vox * r.skip.coutp);
      bf16* xb = role<bf16>(1, wide);
      if (!dry) VRET(ck(vae_cast_bf16(X, static_cast<long long>(vox) * cp, xb, s), "cast"));
      VRET(conv(r.skip, xb, T, H, W, cp, S, CONV_OUT_F32));
      resid = S;
      ready = -1;
    }
    int in = ready;  // norm1(x): fused by the producer of X, else a stand-alone pass into role 1
    if (in < 0) {
      in = 1;
      if (!dry)
        VRET(ck(vae_rmsnorm_silu(X, nullptr, static_cast<long long>(vox), C, cp, r.n1.gamma, role<bf16>(1, wide), s),
                "norm1"));
    }
    int ra = in, rb = 3 - in;  // conv1 reads role ra; conv2 reads role rb (norm2 output)
    bf16* A = role<bf16>(ra, wide);
    bf16* B = role<bf16>(rb, wide);
    if (fusable(r.c1.coutp)) {  // conv1's epilogue writes SiLU(norm2(h)) directly; h is never stored
      VRET(conv(r.c1, A, T, H, W, cp, nullptr, CONV_OUT_NONE, nullptr, false, 0, 0, &r.n2, B));
    } else {
      VRET(conv(r.c1, A, T, H, W, cp, B, CONV_OUT_BF16));
      if (!dry)
        VRET(ck(vae_rmsnorm_silu(nullptr, B, static_cast<long long>(vox), r.c1.cout, r.c1.coutp, r.n2.gamma, A, s),
                "norm2"));
      std::swap(A, B);  // conv2 reads the norm output
      std::swap(ra, rb);
    }
    // x' = x + conv2(...) in the epilogue, fp32, in place over X when the widths agree (each thread
    // reads its own residual element before writing it); the next norm into the buffer conv2 does not read
    const bool fuse_next = next && fusable(r.c2.coutp);
    VRET(conv(r.c2, B, T, H, W, r.c1.coutp, X, CONV_OUT_F32, resid, true, 0, 0, fuse_next ? next : nullptr,
              fuse_next ? A : nullptr));
    ready = fuse_next ? ra : -1;
    C = r.c2.cout;
    cp = r.c2.coutp;
    return GS_OK;
  }
  // the norm the consumer after block b of stage list `blocks` applies to its output
  const VaeNorm* next_norm(const std::vector<VaeRes>& blocks, size_t b, const VaeNorm* after) const {
    if (b + 1 < blocks.size()) return blocks[b + 1].skip.cout ? nullptr : &blocks[b + 1].n1;
    return after;
  }
  int run(const float* lat_dev, int F, int Ht, int Wt, float* video_dev) {
    int T = F, H = 2 * Ht, W = 2 * Wt;
    size_t vox = static_cast<size_t>(T) * H * W;
    bf16* z = role<bf16>(2, vox * v->post.cp);
    if (!dry) VRET(ck(vae_unpatchify(lat_dev, F, Ht, Wt, v->mean, v->stdv, z, v->post.cp, s), "unpatchify"));
    bf16* N = role<bf16>(1, vox * v->post.coutp);
    VRET(conv(v->post, z, T, H, W, v->post.cp, N, CONV_OUT_BF16));
    VRET(conv(v->conv_in, N, T, H, W, v->post.coutp, role<float>(0, vox * v->conv_in.coutp), CONV_OUT_F32));
    int C = v->conv_in.cout, cp = v->conv_in.coutp;
    ready = -1;
    // first block of up stage i (its norm1 can be fused into the stage's entry conv), or null
    auto first_n1 = [&](size_t i) -> const VaeNorm* {
      if (i >= v->up.size() || v->up[i].empty() || v->up[i][0].skip.cout) return nullptr;
      return &v->up[i][0].n1;
    };
    for (size_t b = 0; b < v->mid.size(); ++b)
      VRET(res(v->mid[b], T, H, W, C, cp, next_norm(v->mid, b, first_n1(0))));
    for (size_t i = 0; i < v->up.size(); ++i) {
      const bool last = i + 1 == v->up.size();
      const bool resample = i < v->sconv.size() && v->sconv[i].cout;  // X is read raw (cast / upsample) next
      for (size_t b = 0; b < v->up[i].size(); ++b)
        VRET(res(v->up[i][b], T, H, W, C, cp,
                 next_norm(v->up[i], b, last ? &v->norm_out : (resample ? nullptr : first_n1(i + 1)))));
      if (!resample) continue;
      vox = static_cast<size_t>(T) * H * W;
      bf16* up = nullptr;
      if (v->tconv[i].cout) {  // temporal x2 (reading V5): frame 0 kept, time-conv of frames 1..T-1
        const int T2 = 1 + 2 * (T - 1);
        const size_t fr = static_cast<size_t>(H) * W * cp;
        bf16* xb = role<bf16>(1, vox * cp);
        bf16* tb = role<bf16>(2, fr * T2);
        if (!dry) {
          VRET(ck(vae_cast_bf16(role<float>(0, 0), static_cast<long long>(vox) * cp, xb, s), "cast"));
          VRET(ck(cudaMemcpyAsync(tb, xb, fr * 2, cudaMemcpyDeviceToDevice, s), "frame 0"));
        }
        if (T > 1) VRET(conv(v->tconv[i], xb + fr, T - 1, H, W, cp, tb, CONV_OUT_TIME_INTERLEAVE, nullptr, false, C, cp));
        T = T2;
        up = role<bf16>(1, static_cast<size_t>(T) * 4 * H * W * cp);
        if (!dry) VRET(ck(vae_upsample2(nullptr, tb, T, H, W, cp, up, s), "upsample"));
      } else {
        up = role<bf16>(1, vox * 4 * cp);
        if (!dry) VRET(ck(vae_upsample2(role<float>(0, 0), nullptr, T, H, W, cp, up, s), "upsample"));
      }
      H *= 2;
      W *= 2;
      vox = static_cast<size_t>(T) * H * W;
      // the upsampled input is role 1; the next block's norm1 (fused) goes to role 2
      const VaeNorm* nn = fusable(v->sconv[i].coutp) ? first_n1(i + 1) : nullptr;
      VRET(conv(v->sconv[i], up, T, H, W, cp, role<float>(0, vox * v->sconv[i].coutp), CONV_OUT_F32, nullptr,
                false, 0, 0, nn, nn ? role<bf16>(2, vox * v->sconv[i].coutp) : nullptr));
      ready = nn ? 2 : -1;
      C = v->sconv[i].cout;
      cp = v->sconv[i].coutp;
    }
    vox = static_cast<size_t>(T) * H * W;
    bf16* n = nullptr;
    if (ready > 0) {  // norm_out fused into the last block's conv2
      n = role<bf16>(ready, vox * cp);
    } else {
      n = role<bf16>(1, vox * cp);
      if (!dry) VRET(ck(vae_rmsnorm_silu(role<float>(0, 0), nullptr, static_cast<long long>(vox), C, cp,
                                         v->norm_out.gamma, n, s), "norm_out"));
    }
    ready = -1;
    VRET(conv(v->conv_out, n, T, H, W, cp, video_dev, CONV_OUT_F32_CLAMP, nullptr, false, v->conv_out.cout));
    out_T = T;
    out_H = H;
    out_W = W;
    return GS_OK;
  }
  int out_T = 0, out_H = 0, out_W = 0;
};

int vae_decode_impl(gs_ctx* c, Vae* v, int rank, const float* latent, int F, int Ht, int Wt, float* video,
                    int flags) {
  const int li = vlocal(c, rank);
  if (li < 0) return vfail(c, GS_EINVAL, "rank %d not owned by this process", rank);
  cudaStream_t s = tl_stream ? tl_stream : c->lanes[li];
  if (F < 1 || Ht < 1 || Wt < 1) return vfail(c, GS_EINVAL, "bad latent grid %d x %d x %d", F, Ht, Wt);
  Decoder sizing{c, v, s, true};
  VRET(sizing.run(nullptr, F, Ht, Wt, nullptr));
  const size_t n_lat = static_cast<size_t>(F) * Ht * Wt * 64;
  const size_t n_vid = static_cast<size_t>(sizing.out_T) * sizing.out_H * sizing.out_W * v->desc.out_ch;
  Decoder d{c, v, s, false};
  // grow-only buffers kept in the VAE object (re-used by the next decode on this context)
  auto grow = [&](DevBuf& b, size_t bytes, bool zero) -> int {
    if (b.cap >= bytes) return GS_OK;
    if (b.p) {
      cudaStreamSynchronize(s);
      cudaFree(b.p);
      b.p = nullptr;
      b.cap = 0;
    }
    if (cudaMalloc(&b.p, bytes) != cudaSuccess) {
      cudaGetLastError();
      return vfail(c, GS_ENOMEM, "VAE buffer (%zu B) failed", bytes);
    }
    b.cap = bytes;
    if (zero && cudaMemsetAsync(b.p, 0, bytes, s) != cudaSuccess) return vfail(c, GS_ECUDA, "memset");
    return GS_OK;
  };
  int rc = GS_OK;
  for (int r = 0; r < 4 && rc == GS_OK; ++r) {
    rc = grow(v->act[r], std::max<size_t>(sizing.need[r], 64) * Decoder::esize(r), true);
    d.buf[r] = v->act[r].p;
  }
  const float* lat_dev = latent;
  float* vid_dev = video;
  if (rc == GS_OK && !(flags & 1)) {
    rc = grow(v->lat_stage, n_lat * 4, false);
    if (rc == GS_OK && cudaMemcpyAsync(v->lat_stage.p, latent, n_lat * 4, cudaMemcpyHostToDevice, s) != cudaSuccess)
      rc = vfail(c, GS_ECUDA, "latent upload");
    lat_dev = v->lat_stage.as<float>();
  }
  if (rc == GS_OK && !(flags & 2)) {
    rc = grow(v->vid_stage, n_vid * 4, false);
    vid_dev = v->vid_stage.as<float>();
  }
  if (rc == GS_OK) rc = d.run(lat_dev, F, Ht, Wt, vid_dev);
  if (rc == GS_OK && !(flags & 2) &&
      cudaMemcpyAsync(video, vid_dev, n_vid * 4, cudaMemcpyDeviceToHost, s) != cudaSuccess)
    rc = vfail(c, GS_ECUDA, "video download");
  cudaError_t e = cudaStreamSynchronize(s);
  if (rc == GS_OK && e != cudaSuccess) rc = vfail(c, GS_ECUDA, "VAE decode: %s", cudaGetErrorString(e));
  return rc;
}

}  // namespace

extern "C" {

int gs_vae_create(gs_ctx* c, const gs_vae_desc* d, int* vae_id) {
  if (!c || !d || !vae_id) return GS_EINVAL;
  std::lock_guard<std::mutex> g(c->api_mu);
  {
    std::lock_guard<std::mutex> g2(c->table_mu);
    if (!c->tickets.empty()) return vfail(c, GS_ESTATE, "gs_vae_create needs every run waited for");
  }
  VCK(cudaSetDevice(c->device));
  if (d->z_dim != 16 || d->out_ch < 1 || d->out_ch > 64 || d->blocks < 1 || d->mid_blocks < 0)
    return vfail(c, GS_EINVAL, "unsupported VAE shape (z_dim %d out %d)", d->z_dim, d->out_ch);
  for (int i = 0; i < 5; ++i)
    if (d->dims[i] < 64 || d->dims[i] % 64 != 0 && d->dims[i] % 32 != 0 || d->dims[i] > 512)
      return vfail(c, GS_EINVAL, "VAE width %d unsupported (multiple of 32, 64..512)", d->dims[i]);
  auto v = std::make_unique<Vae>();
  v->desc = *d;
  Gen gen{c, v.get(), c->stream};
  auto cleanup = [&](int rc) {
    cudaStreamSynchronize(c->stream);
    for (void* p : v->allocs) cudaFree(p);
    return rc;
  };
  // module 0: latent statistics (mean = 0.5 u, std = 1 + 0.25 u; fp32 as synth/vae.py)
  int rc = GS_OK;
  void *mean = nullptr, *stdv = nullptr;
  if ((rc = gen.alloc(&mean, 16 * 4)) != GS_OK || (rc = gen.alloc(&stdv, 16 * 4)) != GS_OK) return cleanup(rc);
  float hstd[16];
  if (rng_fill(mean, 16, d->weight_seed, 200, RNG_F32_SCALED, 0.5f, c->stream) != cudaSuccess ||
      rng_fill(stdv, 16, d->weight_seed, 201, RNG_F32_SCALED, 0.25f, c->stream) != cudaSuccess ||
      cudaMemcpyAsync(hstd, stdv, 64, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
      cudaStreamSynchronize(c->stream) != cudaSuccess)
    return cleanup(vfail(c, GS_ECUDA, "VAE statistics"));
  for (float& x : hstd) x = 1.0f + x;  // one IEEE fp32 add, as numpy's float32(1) + float32(0.25 u)
  if (cudaMemcpy(stdv, hstd, 64, cudaMemcpyHostToDevice) != cudaSuccess)
    return cleanup(vfail(c, GS_ECUDA, "VAE statistics upload"));
  v->mean = static_cast<float*>(mean);
  v->stdv = static_cast<float*>(stdv);
  gen.module = 1;
  const int* dm = d->dims;
  if ((rc = gen.conv(v->post, d->z_dim, d->z_dim, 1, 1, 1)) != GS_OK) return cleanup(rc);
  if ((rc = gen.conv(v->conv_in, d->z_dim, dm[0], 3, 3, 3)) != GS_OK) return cleanup(rc);
  v->mid.resize(d->mid_blocks);
  for (VaeRes& r : v->mid)
    if ((rc = gen.res(r, dm[0], dm[0])) != GS_OK) return cleanup(rc);
  const int nst = 4;
  v->up.resize(nst);
  v->tconv.resize(nst);
  v->sconv.resize(nst);
  int cin = dm[0];
  for (int i = 0; i < nst; ++i) {
    const int cout = dm[i + 1];
    if (i >= 1) cin = dm[i] / 2;
    v->up[i].resize(d->blocks);
    for (VaeRes& r : v->up[i]) {
      if ((rc = gen.res(r, cin, cout)) != GS_OK) return cleanup(rc);
      cin = cout;
    }
    if (i < nst - 1) {
      if (d->temporal_up[i] && (rc = gen.conv(v->tconv[i], cout, 2 * cout, 3, 1, 1)) != GS_OK) return cleanup(rc);
      if ((rc = gen.conv(v->sconv[i], cout, cout / 2, 1, 3, 3)) != GS_OK) return cleanup(rc);
    }
  }
  if ((rc = gen.norm(v->norm_out, dm[4])) != GS_OK) return cleanup(rc);
  if ((rc = gen.conv(v->conv_out, dm[4], d->out_ch, 3, 3, 3)) != GS_OK) return cleanup(rc);
  VCK(cudaStreamSynchronize(c->stream));
  *vae_id = static_cast<int>(c->vaes.size());
  c->vaes.push_back(std::move(v));
  return GS_OK;
}

int gs_vae_decode(gs_ctx* c, int vae_id, int rank, const float* latent, int F, int Ht, int Wt, float* video,
                  int flags) {
  if (!c || !latent || !video) return GS_EINVAL;
  std::lock_guard<std::mutex> g(c->api_mu);
  VCK(cudaSetDevice(c->device));
  if (vae_id < 0 || vae_id >= static_cast<int>(c->vaes.size())) return vfail(c, GS_EINVAL, "bad VAE id");
  {
    std::lock_guard<std::mutex> g2(c->table_mu);
    if (rank >= 0 && rank < c->world && c->busy[rank])
      return vfail(c, GS_ESTATE, "rank %d belongs to in-flight run %llu", rank, (unsigned long long)c->busy[rank]);
  }
  return vae_decode_impl(c, c->vaes[vae_id].get(), rank, latent, F, Ht, Wt, video, flags);
}

int gs_vae_decode_request(gs_ctx* c, int vae_id, gs_req id, float* video) {
  if (!c || !video) return GS_EINVAL;
  Request* q = nullptr;
  {
    std::lock_guard<std::mutex> g(c->table_mu);
    auto it = c->reqs.find(id);
    if (it == c->reqs.end()) return vfail(c, GS_EINVAL, "unknown request");
    q = it->second.get();
    if (q->state == GS_REQ_RUNNING || q->state == GS_REQ_QUEUED)
      return vfail(c, GS_ESTATE, "request is %s", q->state == GS_REQ_RUNNING ? "running" : "queued");
    for (const Shard& s : q->shards)
      if (vlocal(c, s.rank) < 0) return vfail(c, GS_EUNSUPPORTED, "shard on rank %d is not in this process", s.rank);
  }
  VCK(cudaSetDevice(c->device));
  const int rank = q->ranks[0];
  cudaStream_t s = c->lanes[vlocal(c, rank)];
  const size_t lat = 64;
  float* dev = nullptr;
  if (cudaMalloc(&dev, static_cast<size_t>(q->n) * lat * 4) != cudaSuccess) {
    cudaGetLastError();
    return vfail(c, GS_ENOMEM, "latent gather");
  }
  int rc = GS_OK;
  for (const Shard& sh : q->shards)  // contiguous token ranges -> one latent on the decoding GPU
    if (sh.z && sh.hi > sh.lo &&
        cudaMemcpyAsync(dev + static_cast<size_t>(sh.lo) * lat, sh.z, static_cast<size_t>(sh.hi - sh.lo) * lat * 4,
                        cudaMemcpyDeviceToDevice, s) != cudaSuccess)
      rc = vfail(c, GS_ECUDA, "latent gather copy");
  if (rc == GS_OK) rc = gs_vae_decode(c, vae_id, rank, dev, q->grid[0], q->grid[1], q->grid[2], video, 1);
  cudaStreamSynchronize(s);
  cudaFree(dev);
  return rc;
}

int gs_debug_conv3d(gs_ctx* c, const void* x, const void* w, const void* bias, const void* resid, void* out, int T,
                    int H, int W, int Cp, int kt, int kh, int kw, int Coutp, int out_cs, int mode, int out_real) {
  if (!c || !x || !w || !bias || !out) return GS_EINVAL;
  std::lock_guard<std::mutex> g(c->api_mu);
  VCK(cudaSetDevice(c->device));
  ConvParams p{T, H, W, Cp, kt, kh, kw, Coutp, static_cast<const bf16*>(bias), static_cast<const bf16*>(resid),
               out, out_cs, mode, out_real};
  cudaEvent_t ev;
  VCK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  VCK(cudaEventRecord(ev, cudaStreamLegacy));  // caller's buffers come from the legacy stream (torch)
  VCK(cudaStreamWaitEvent(c->stream, ev, 0));
  cudaEventDestroy(ev);
  cudaError_t e = conv3d_tc(x, w, p, c->num_sms, c->stream);
  if (e != cudaSuccess) return vfail(c, e == cudaErrorInvalidValue ? GS_EINVAL : GS_ECUDA, "conv3d: %s",
                                     cudaGetErrorString(e));
  VCK(cudaStreamSynchronize(c->stream));
  return GS_OK;
}

}  // extern "C"
