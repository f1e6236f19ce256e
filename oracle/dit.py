"""fp64 CPU oracle of the GenServe DiT-step hot path.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
cpu_baseline / `--impl reference` leg may import this module.  The product path
(`paper_2604_04335_b200`) never imports, calls or links anything under `oracle/`, and
this file shares no code with it (only the seeded input generators in `synth/`).

What it computes.  The paper (PAPER.md, arxiv 2604.04335) serves DiT models whose
reverse diffusion step (§2.1, Eq. "reverse process") is one DiT forward
("DiT blocks that perform N denoising steps", §2.1) followed by a sampler update.
It does not spell out the block; the readings below are SURVEY.md §8(c) readings 1-16,
restated in DESIGN.md "Readings".  Everything is a plain definition written out in fp64
numpy; the only library primitives are matmul/einsum, exp, tanh, sqrt, sin, cos.

Block (SURVEY.md §8(c) "Block"), per layer, r(i) = request of row i,
e_r = M_l + e(t_r) in R^{6 x D} split (sh1, sc1, g1, sh2, sc2, g2):
  1. a  = LN(x) * (1 + sc1) + sh1              LN: biased var, eps 1e-6, no affine
  2. q,k,v = a W_{q,k,v}^T + b
  3. q <- q / sqrt(mean_D q^2 + eps) * g_q      (RMSNorm over the full D); same for k
  4. RoPE on q, k per head, 3 axes (f, h, w), pair slots [d/2-2*floor(d/6), floor(d/6), floor(d/6)]
  5. O_h = softmax(q_h k_h^T / sqrt(d)) v_h      over the request's own tokens only
  6. x <- x + g1 * (O W_o^T + b_o)
  7. x <- x + g2 * (GELU_tanh(LN(x)(1+sc2)+sh2) W_1^T + b_1) W_2^T + b_2)
Step (SURVEY.md §8(c) "Step"): x = z W_pe^T + b_pe; e0 = time MLP of t = 1000 sigma;
e = W_p SiLU(e0) + b_p; L blocks; head v = (LN(x)(1+hsc)+hsh) W_head^T + b_head with
(hsh, hsc) = M_head + e0; Euler z <- z + (sigma_{i+1} - sigma_i) v;
sigma_i = s u_i / (1 + (s-1) u_i), u_i = 1 - i/S, s = 5 (FlowMatch Euler, reading 5).

Text cross-attention + CFG (the paper's blocks have cross-attention,
P:135 §2.1, and its VideoState carries prompt embeddings, P:759 / Tab. paused_memory; DESIGN.md
readings 19-21): after the self-attention residual,
  x <- x + (softmax(q k^T / sqrt d) v) W_co^T + b_co,  q = RMS(LN_aff(x) W_cq^T + b_cq) g_cq,
  [k|v] = c W_ckv^T + b_ckv, k <- RMS(k) g_ck,  c = W_te2 GELU_tanh(W_te1 emb + b) + b,
with LN_aff = LN(x) * ln3_w + ln3_b (no modulation, no gate, no RoPE); classifier-free guidance
v = v_u + g (v_c - v_u) from the forwards with the cond / uncond prompt embeddings.

Parity pins: tests/test_oracle_pins.py (brute force, closed forms, invariants, the
paper's Tab.3 cost model).  Parity unpinned: agreement with the *trained* Wan/SD3.5
models (no trained weights exist here).
"""
import math

import numpy as np

EPS = 1e-6
ROPE_THETA = 10000.0


# --------------------------------------------------------------------------------------
# components
# --------------------------------------------------------------------------------------
def layer_norm(x, eps=EPS):
    """LN without affine, biased variance (reading 1; Wan LayerNorm(elementwise_affine=False))."""
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + eps)


def modulate(a, shift, scale):
    """adaLN modulation a*(1+scale)+shift (block step 1 / 7, reading 1)."""
    return a * (1.0 + scale) + shift


def rms_norm(x, g, eps=EPS):
    """RMSNorm over the last axis (the full model dim D for q/k, reading 1)."""
    return x / np.sqrt((x * x).mean(axis=-1, keepdims=True) + eps) * g


def gelu_tanh(u):
    """GELU, tanh approximation: 0.5u(1+tanh(sqrt(2/pi)(u+0.044715u^3)))."""
    return 0.5 * u * (1.0 + np.tanh(math.sqrt(2.0 / math.pi) * (u + 0.044715 * u ** 3)))


def silu(u):
    return u / (1.0 + np.exp(-u))


def linear(x, w, b=None):
    """x W^T + b (PyTorch nn.Linear convention, W: [out, in])."""
    y = x @ w.T
    return y if b is None else y + b


def rope_slots(d):
    """Pair slots per axis (f, h, w): [d/2 - 2*floor(d/6), floor(d/6), floor(d/6)]."""
    s = d // 6
    return (d // 2 - 2 * s, s, s)


def token_positions(grid):
    """(f, h, w) position of each request-local token index i in (f, h, w) row order."""
    F, H, W = grid
    i = np.arange(F * H * W)
    return np.stack([i // (H * W), (i // W) % H, i % W], axis=1)


def _positions(grid_or_pos):
    if isinstance(grid_or_pos, np.ndarray):
        return grid_or_pos
    return token_positions(grid_or_pos)


def rope_angles(pos, d, theta=ROPE_THETA):
    """Angles [n, d/2]: slot j of axis a (width m_a = 2*slots_a) gets pos_a * theta^(-2j/m_a)."""
    cols = []
    for a, slots in enumerate(rope_slots(d)):
        m = 2 * slots
        inv = theta ** (-2.0 * np.arange(slots) / m)
        cols.append(np.outer(pos[:, a].astype(np.float64), inv))
    return np.concatenate(cols, axis=1)


def rope_apply(x, ang):
    """Rotate consecutive pairs (2j, 2j+1) of x [n, H, d] by ang [n, d/2] (complex multiply)."""
    c = np.cos(ang)[:, None, :]
    s = np.sin(ang)[:, None, :]
    x0 = x[..., 0::2]
    x1 = x[..., 1::2]
    out = np.empty_like(x)
    out[..., 0::2] = x0 * c - x1 * s
    out[..., 1::2] = x0 * s + x1 * c
    return out


def softmax(s, axis=-1):
    s = s - s.max(axis=axis, keepdims=True)
    p = np.exp(s)
    return p / p.sum(axis=axis, keepdims=True)


def attention(q, k, v):
    """Full non-causal attention of one request: q [nq, H, d], k/v [n, H, d] -> [nq, H, d]."""
    d = q.shape[-1]
    s = np.matmul(q.transpose(1, 0, 2), k.transpose(1, 2, 0)) / math.sqrt(d)   # [H, nq, n]
    p = softmax(s, axis=-1)
    return np.matmul(p, v.transpose(1, 0, 2)).transpose(1, 0, 2)              # [nq, H, d]


# --------------------------------------------------------------------------------------
# text cross-attention (NEXT-1)
# --------------------------------------------------------------------------------------
def text_embedding(emb, glob):
    """c = W_te2 GELU_tanh(W_te1 emb + b_te1) + b_te2 for prompt embeddings emb [L, text_dim]."""
    return linear(gelu_tanh(linear(emb, glob["w_te1"], glob["b_te1"])), glob["w_te2"], glob["b_te2"])


def layer_norm_affine(x, w, b, eps=EPS):
    """LN with elementwise affine (Wan norm3, cross_attn_norm=True [ext])."""
    return layer_norm(x, eps) * w + b


def cross_kv(c, blk, heads):
    """Per-layer context keys / values of one prompt: k = RMS(c W_ck^T + b) g_ck, v = c W_cv^T + b."""
    L, D = c.shape
    kv = linear(c, blk["w_ckv"], blk["b_ckv"])
    k = rms_norm(kv[:, :D], blk["g_ck"])
    return k.reshape(L, heads, D // heads), kv[:, D:].reshape(L, heads, D // heads)


def cross_attention(x, blk, c, heads):
    """Cross-attention branch of rows x [n, D] of one request branch against its context c."""
    n, D = x.shape
    d = D // heads
    a = layer_norm_affine(x, blk["ln3_w"], blk["ln3_b"])
    q = rms_norm(linear(a, blk["w_cq"], blk["b_cq"]), blk["g_cq"]).reshape(n, heads, d)
    k, v = cross_kv(c, blk, heads)
    return linear(attention(q, k, v).reshape(n, D), blk["w_co"], blk["b_co"])


# --------------------------------------------------------------------------------------
# block
# --------------------------------------------------------------------------------------
def _split_mod(mod_rows):
    return [mod_rows[:, c, :] for c in range(6)]


def dit_block(x, blk, e_req, reqs, heads, ctxs=None):
    """One DiT block over a varlen-packed batch.

    x      [N, D] fp64, rows of the requests concatenated in `reqs` order
    blk    dict of fp64 params (see synth.block_params)
    e_req  [B, 6, D] time-embedding projection e(t_r) per request (M_l added here)
    reqs   list of (offset, n, grid_or_pos) per request; grid = (F_lat, H_t, W_t) or an
           explicit [n, 3] int array of (f, h, w) RoPE positions
    ctxs   (cross-attention models) per-request text context c [L, D] (text_embedding output)
    """
    N, D = x.shape
    d = D // heads
    row_req = np.empty(N, dtype=np.int64)
    for r, (off, n, _g) in enumerate(reqs):
        row_req[off:off + n] = r
    mod = blk["mod"][None, :, :] + e_req[row_req]        # [N, 6, D]
    sh1, sc1, g1, sh2, sc2, g2 = _split_mod(mod)

    a = modulate(layer_norm(x), sh1, sc1)
    qkv = linear(a, blk["w_qkv"], blk["b_qkv"])
    q, k, v = qkv[:, :D], qkv[:, D:2 * D], qkv[:, 2 * D:]
    q = rms_norm(q, blk["g_q"])
    k = rms_norm(k, blk["g_k"])
    o = np.empty((N, heads, d))
    for off, n, grid in reqs:
        ang = rope_angles(_positions(grid), d)
        qh = rope_apply(q[off:off + n].reshape(n, heads, d), ang)
        kh = rope_apply(k[off:off + n].reshape(n, heads, d), ang)
        vh = v[off:off + n].reshape(n, heads, d)
        o[off:off + n] = attention(qh, kh, vh)
    x = x + g1 * linear(o.reshape(N, D), blk["w_o"], blk["b_o"])
    if ctxs is not None:
        for (off, n, _g), c in zip(reqs, ctxs):
            x[off:off + n] = x[off:off + n] + cross_attention(x[off:off + n], blk, c, heads)
    a2 = modulate(layer_norm(x), sh2, sc2)
    h = gelu_tanh(linear(a2, blk["w_1"], blk["b_1"]))
    return x + g2 * linear(h, blk["w_2"], blk["b_2"])


def dit_block_rows(x, blk, e, grid, heads, rows, ctx=None):
    """Row-sampled DiT block of ONE request (SURVEY.md §8(c) 'Large configs').

    Computes LN1 and K/V for all n tokens, everything else only for `rows`.
    Returns x_out[rows] — identical (same fp64 formula) to dit_block(...)[rows].
    """
    n, D = x.shape
    d = D // heads
    rows = np.asarray(rows)
    mod = blk["mod"] + e                                  # [6, D]
    sh1, sc1, g1, sh2, sc2, g2 = (mod[c] for c in range(6))
    a = modulate(layer_norm(x), sh1, sc1)
    wq, wk, wv = (blk["w_qkv"][i * D:(i + 1) * D] for i in range(3))
    bq, bk, bv = (blk["b_qkv"][i * D:(i + 1) * D] for i in range(3))
    pos = token_positions(grid)
    k = rms_norm(linear(a, wk, bk), blk["g_k"])
    k = rope_apply(k.reshape(n, heads, d), rope_angles(pos, d))
    v = linear(a, wv, bv).reshape(n, heads, d)
    q = rms_norm(linear(a[rows], wq, bq), blk["g_q"])
    q = rope_apply(q.reshape(len(rows), heads, d), rope_angles(pos[rows], d))
    o = attention(q, k, v).reshape(len(rows), D)
    xr = x[rows] + g1 * linear(o, blk["w_o"], blk["b_o"])
    if ctx is not None:
        xr = xr + cross_attention(xr, blk, ctx, heads)
    a2 = modulate(layer_norm(xr), sh2, sc2)
    return xr + g2 * linear(gelu_tanh(linear(a2, blk["w_1"], blk["b_1"])), blk["w_2"], blk["b_2"])


# --------------------------------------------------------------------------------------
# step
# --------------------------------------------------------------------------------------
def sigmas(steps, shift=5.0):
    """FlowMatch shifted schedule sigma_i = s u/(1+(s-1)u), u = 1 - i/S, i = 0..S (reading 5)."""
    u = 1.0 - np.arange(steps + 1, dtype=np.float64) / steps
    return shift * u / (1.0 + (shift - 1.0) * u)


def sinusoid(t, freq_dim=256):
    """[cos(t w_j), sin(t w_j)], w_j = 10000^(-j/half), j < half (Wan sinusoidal_embedding_1d)."""
    half = freq_dim // 2
    w = 10000.0 ** (-np.arange(half, dtype=np.float64) / half)
    return np.concatenate([np.cos(t * w), np.sin(t * w)])


def time_embedding(t, glob):
    """e0 = W_t2 SiLU(W_t1 s(t) + b) + b;  e = W_tp SiLU(e0) + b_tp reshaped [6, D]."""
    s = sinusoid(t, glob["w_t1"].shape[1])
    e0 = linear(silu(linear(s, glob["w_t1"], glob["b_t1"])), glob["w_t2"], glob["b_t2"])
    e = linear(silu(e0), glob["w_tp"], glob["b_tp"]).reshape(6, -1)
    return e0, e


def patch_embed(z, glob):
    """x = z W_pe^T + b_pe for token-major latent z [n, 64] (patchify is the identity here:
    the synthetic latent is generated token-major)."""
    return linear(z, glob["w_pe"], glob["b_pe"])


def head(x, e0_rows, glob):
    """v = (LN(x)(1+hsc)+hsh) W_head^T + b_head, (hsh, hsc) = M_head + e0."""
    hsh = glob["mod_head"][0] + e0_rows
    hsc = glob["mod_head"][1] + e0_rows
    return linear(modulate(layer_norm(x), hsh, hsc), glob["w_head"], glob["b_head"])


def euler(z, v, sig_i, sig_next):
    """z <- z + (sigma_{i+1} - sigma_i) v."""
    return z + (sig_next - sig_i) * v


def dit_velocity(z_list, grids, ts, glob, blocks, heads, ctxs=None):
    """DiT forward of a batch: z_list[r] [n_r, 64], t_r (and text context c_r) -> velocity list."""
    offs, reqs = 0, []
    for z, g in zip(z_list, grids):
        reqs.append((offs, z.shape[0], g))
        offs += z.shape[0]
    z = np.concatenate(z_list, axis=0)
    x = patch_embed(z, glob)
    e0s, es = zip(*(time_embedding(t, glob) for t in ts))
    e_req = np.stack(es)
    for blk in blocks:
        x = dit_block(x, blk, e_req, reqs, heads, ctxs)
    e0_rows = np.concatenate([np.broadcast_to(e0s[r], (n, e0s[r].shape[0]))
                              for r, (_o, n, _g) in enumerate(reqs)])
    v = head(x, e0_rows, glob)
    return [v[o:o + n] for o, n, _g in reqs]


def cfg_velocity(v_cond, v_uncond, g):
    """Classifier-free guidance v = v_u + g (v_c - v_u) (reading 21)."""
    return v_uncond + g * (v_cond - v_uncond)


def dit_steps(z_list, grids, step_idx, n_steps, k, glob, blocks, heads, shift=5.0, prompts=None,
              cfg=None):
    """Run k denoising steps of a batch; request r is at step index step_idx[r] of n_steps.

    prompts[r] = (emb_cond, emb_uncond or None) prompt embeddings (cross-attention models);
    cfg[r] = guidance scale g_r (CFG when emb_uncond is given)."""
    z_list = [np.asarray(z, dtype=np.float64) for z in z_list]
    sig = sigmas(n_steps, shift)
    step_idx = list(step_idx)
    ctx_c = ctx_u = None
    if prompts is not None:
        ctx_c = [text_embedding(pc, glob) for pc, _pu in prompts]
        ctx_u = [None if pu is None else text_embedding(pu, glob) for _pc, pu in prompts]
    for _ in range(k):
        ts = [1000.0 * sig[i] for i in step_idx]
        vs = dit_velocity(z_list, grids, ts, glob, blocks, heads, ctx_c)
        if ctx_u is not None and any(c is not None for c in ctx_u):
            for r, cu in enumerate(ctx_u):
                if cu is not None:
                    vu = dit_velocity([z_list[r]], [grids[r]], [ts[r]], glob, blocks, heads, [cu])[0]
                    vs[r] = cfg_velocity(vs[r], vu, cfg[r])
        z_list = [euler(z, v, sig[i], sig[i + 1]) for z, v, i in zip(z_list, vs, step_idx)]
        step_idx = [i + 1 for i in step_idx]
    return z_list
