"""fp64 CPU oracle of the VAE decode stage.

TEST INFRASTRUCTURE ONLY (see oracle/dit.py header): importable from tests/, smoke() and bench.py's
cpu_baseline leg; the product path never imports it, and it shares no code with csrc/vae.cpp.

What it computes.  The paper's pipeline ends with "a VAE for latent encoding/decoding" (§2.1)
whose decode runs on a single GPU, decoupled from the DiT (§4.3; Tab. stage_breakdown
P:186-194: 5-8% of e2e).  The paper gives no VAE internals.  Readings:
  V1 the decoder is Wan2.1-VAE-shaped [ext]: widths (384, 384, 384, 192, 96), causal 3-D convs,
     residual blocks, x4 temporal / x8 spatial upsampling (synth/vae.py module walk);
  V2 CausalConv3d(kt, kh, kw): zero padding of kt - 1 frames BEFORE the sequence (none after) and
     (kh - 1) / 2, (kw - 1) / 2 on both sides in H, W; stride 1;
  V3 RMS norm over channels as Wan's RMS_norm: x * sqrt(C) / max(||x||_2, 1e-12) * gamma (no bias);
  V4 no mid attention block (Wan's single-head spatial attention at the lowest resolution, ~2% of
     the decoder FLOPs at 720p) -- out of scope;
  V5 upsample3d(C): time_conv (3,1,1) C -> 2C over frames 1..T-1 only (frame 0 is not in its causal
     history: Wan's first-chunk 'Rep' cache), output frames [x_0, y_1[:C], y_1[C:], y_2[:C], ...]
     (T -> 1 + 2 (T - 1)); then nearest x2 in H, W and a (1,3,3) conv C -> C/2 on every frame;
     upsample2d(C): nearest x2 in H, W and a (1,3,3) conv C -> C/2;
  V6 input: the DiT latent [n, 64] (token-major, (f, h, w) rows, feature order (c, pt, ph, pw),
     DiT patch (1, 2, 2)) unpatchified to z [F, 2 H_t, 2 W_t, 16], de-normalised z * std + mean per
     channel (Wan's latent statistics; synthetic seeded values here), then a 1x1x1 conv 16 -> 16;
  V7 output: conv_out of SiLU(RMS(x)), clamped to [-1, 1]: video [T_out, 16 H_t, 16 W_t, 3];
  V8 activations channels-last [T, H, W, C].
Only library primitive: matmul (one per conv tap); everything else is written out.
Parity pins: tests/test_vae_pins.py.
"""
import numpy as np

from synth.rng import bf16_bits_to_f64


def _f64(a):
    return bf16_bits_to_f64(a) if a.dtype == np.uint16 else np.asarray(a, np.float64)


def causal_conv3d(x, w, b):
    """x [T, H, W, Cin], w [Cout, kt, kh, kw, Cin], b [Cout] -> y [T, H, W, Cout] (reading V2):
    y[t, h, w] = b + sum over taps (dt, dh, dw) of w[:, dt, dh, dw, :] . xpad[t + dt, h + dh, w + dw]."""
    T, H, W, _ = x.shape
    _, kt, kh, kw, _ = w.shape
    ph, pw = (kh - 1) // 2, (kw - 1) // 2
    xp = np.zeros((T + kt - 1, H + 2 * ph, W + 2 * pw, x.shape[3]))
    xp[kt - 1:, ph:ph + H, pw:pw + W] = x
    y = np.broadcast_to(b, (T, H, W, w.shape[0])).copy()
    for dt in range(kt):
        for dh in range(kh):
            for dw in range(kw):
                y += xp[dt:dt + T, dh:dh + H, dw:dw + W] @ w[:, dt, dh, dw, :].T
    return y


def rms_norm_c(x, gamma):
    """Wan RMS_norm over channels (reading V3): x sqrt(C) / max(||x||, 1e-12) gamma."""
    n = np.sqrt((x * x).sum(axis=-1, keepdims=True))
    return x * np.sqrt(x.shape[-1]) / np.maximum(n, 1e-12) * gamma


def silu(x):
    return x / (1.0 + np.exp(-x))


def resblock(x, p, prefix):
    """h = conv1(SiLU(RMS1(x))); h = conv2(SiLU(RMS2(h))); x' = h + x (or skip(x) when widths differ)."""
    h = causal_conv3d(silu(rms_norm_c(x, p[prefix + ".norm1"]["gamma"])), p[prefix + ".conv1"]["w"],
                      p[prefix + ".conv1"]["b"])
    h = causal_conv3d(silu(rms_norm_c(h, p[prefix + ".norm2"]["gamma"])), p[prefix + ".conv2"]["w"],
                      p[prefix + ".conv2"]["b"])
    sk = p.get(prefix + ".skip")
    return h + (causal_conv3d(x, sk["w"], sk["b"]) if sk is not None else x)


def upsample_nearest2(x):
    """Nearest-neighbour x2 in H and W: out[t, h, w] = x[t, h // 2, w // 2]."""
    return x.repeat(2, axis=1).repeat(2, axis=2)


def temporal_upsample(x, w, b):
    """Reading V5: time_conv over frames 1..T-1, each giving two output frames; frame 0 kept."""
    C = x.shape[-1]
    out = [x[:1]]
    if x.shape[0] > 1:
        y = causal_conv3d(x[1:], w, b)                     # [T - 1, H, W, 2C]
        inter = np.stack([y[..., :C], y[..., C:]], axis=1)   # [T - 1, 2, H, W, C]
        out.append(inter.reshape(-1, *x.shape[1:]))
    return np.concatenate(out, axis=0)


def unpatchify(lat, grid, z_dim=16):
    """DiT latent [n, 64] (rows (f, h, w), features (c, pt, ph, pw), patch (1, 2, 2)) ->
    z [F, 2 H_t, 2 W_t, z_dim] with z[f, 2 h + ph, 2 w + pw, c] = lat[(f, h, w), (c, 0, ph, pw)]
    (reading V6)."""
    F, Ht, Wt = grid
    a = np.asarray(lat, np.float64).reshape(F, Ht, Wt, z_dim, 1, 2, 2)
    z = np.empty((F, 2 * Ht, 2 * Wt, z_dim))
    for ph in range(2):
        for pw in range(2):
            z[:, ph::2, pw::2, :] = a[:, :, :, :, 0, ph, pw]
    return z


def decode(lat, grid, params, shape):
    """The decoder of synth/vae.py's module walk: DiT latent [n, 64] -> video [T_out, H, W, 3]."""
    p = {k: {t: _f64(v) for t, v in d.items()} for k, d in params.items()}
    z = unpatchify(lat, grid, shape.z_dim)
    z = z * p["znorm"]["std"] + p["znorm"]["mean"]
    x = causal_conv3d(z, p["post"]["w"], p["post"]["b"])
    x = causal_conv3d(x, p["conv_in"]["w"], p["conv_in"]["b"])
    for b in range(shape.mid_blocks):
        x = resblock(x, p, f"mid.{b}")
    nst = len(shape.dims) - 1
    for i in range(nst):
        for b in range(shape.blocks):
            x = resblock(x, p, f"up{i}.{b}")
        if i < nst - 1:
            if shape.temporal_up[i]:
                x = temporal_upsample(x, p[f"up{i}.tconv"]["w"], p[f"up{i}.tconv"]["b"])
            x = causal_conv3d(upsample_nearest2(x), p[f"up{i}.sconv"]["w"], p[f"up{i}.sconv"]["b"])
    x = causal_conv3d(silu(rms_norm_c(x, p["norm_out"]["gamma"])), p["conv_out"]["w"], p["conv_out"]["b"])
    return np.clip(x, -1.0, 1.0)


def decode_flops(grid, shape, vae_modules):
    """Multiply-add FLOPs (2 per MAC) of the decoder's convolutions for a latent grid."""
    F, Ht, Wt = grid
    T, H, W = F, 2 * Ht, 2 * Wt
    mods = {m[0]: m for m in vae_modules(shape)}
    tot = 0

    def conv(name, t, h, w):
        _n, _k, cin, cout, (kt, kh, kw) = mods[name]
        return 2 * t * h * w * cout * cin * kt * kh * kw

    tot += conv("post", T, H, W) + conv("conv_in", T, H, W)
    for name in mods:
        if name.startswith("mid.") and (name.endswith(".conv1") or name.endswith(".conv2")):
            tot += conv(name, T, H, W)
    nst = len(shape.dims) - 1
    for i in range(nst):
        for name in mods:
            if name.startswith(f"up{i}.") and name.split(".")[-1] in ("conv1", "conv2", "skip"):
                tot += conv(name, T, H, W)
        if i < nst - 1:
            if shape.temporal_up[i]:
                tot += conv(f"up{i}.tconv", T - 1, H, W)
                T = 1 + 2 * (T - 1)
            H, W = 2 * H, 2 * W
            tot += conv(f"up{i}.sconv", T, H, W)
    tot += conv("conv_out", T, H, W)
    return tot
