"""Pins of the VAE-decode oracle (oracle/vae.py) against brute force, closed
forms and invariants -- nothing here re-types the oracle's formulas."""
import math

import numpy as np
import pytest

from oracle import vae
from synth import vae as sv

RNG = np.random.default_rng(17)


def test_causal_conv3d_brute_force_fsum():
    """Reading V2 written as scalar loops with math.fsum: zero padding of kt-1 frames before the
    sequence only, (k-1)/2 on each side in H and W, w[co, dt, dh, dw, ci] on xpad[t+dt, h+dh, w+dw]."""
    T, H, W, Ci, Co = 3, 3, 4, 2, 3
    for k in [(3, 3, 3), (3, 1, 1), (1, 3, 3), (1, 1, 1)]:
        x = RNG.standard_normal((T, H, W, Ci))
        w = RNG.standard_normal((Co, *k, Ci))
        b = RNG.standard_normal(Co)
        y = vae.causal_conv3d(x, w, b)
        kt, kh, kw = k
        for t in range(T):
            for h in range(H):
                for ww in range(W):
                    for co in range(Co):
                        terms = [b[co]]
                        for dt in range(kt):
                            for dh in range(kh):
                                for dw in range(kw):
                                    ti, hi, wi = t + dt - (kt - 1), h + dh - (kh - 1) // 2, ww + dw - (kw - 1) // 2
                                    if 0 <= ti < T and 0 <= hi < H and 0 <= wi < W:
                                        terms += [w[co, dt, dh, dw, ci] * x[ti, hi, wi, ci] for ci in range(Ci)]
                        assert y[t, h, ww, co] == pytest.approx(math.fsum(terms), abs=1e-12)


def test_conv_is_causal_in_time():
    """Output frame t never depends on input frames > t."""
    x = RNG.standard_normal((5, 4, 4, 3))
    w = RNG.standard_normal((2, 3, 3, 3, 3))
    y0 = vae.causal_conv3d(x, w, np.zeros(2))
    x2 = x.copy()
    x2[3:] += 5.0
    y1 = vae.causal_conv3d(x2, w, np.zeros(2))
    np.testing.assert_array_equal(y0[:3], y1[:3])
    assert not np.allclose(y0[3:], y1[3:])


def test_delta_kernel_is_identity_and_1x1_is_matmul():
    x = RNG.standard_normal((2, 3, 5, 4))
    w = np.zeros((4, 3, 3, 3, 4))
    for c in range(4):
        w[c, 2, 1, 1, c] = 1.0            # current frame, centre pixel
    np.testing.assert_allclose(vae.causal_conv3d(x, w, np.zeros(4)), x, atol=0)
    m = RNG.standard_normal((6, 4))
    np.testing.assert_allclose(vae.causal_conv3d(x, m.reshape(6, 1, 1, 1, 4), np.ones(6)),
                               np.einsum("thwc,oc->thwo", x, m) + 1.0, atol=1e-12)


def test_rms_norm_closed_forms():
    """Reading V3: a constant vector c*1 maps to sign(c)*gamma; the output RMS over channels is
    |gamma| RMS-weighted to sqrt(C)/sqrt(C) = 1 when gamma = 1."""
    g = RNG.uniform(0.9, 1.1, 8)
    np.testing.assert_allclose(vae.rms_norm_c(np.full((1, 8), -3.0), g), -g[None], atol=1e-15)
    x = RNG.standard_normal((5, 8))
    y = vae.rms_norm_c(x, np.ones(8))
    np.testing.assert_allclose(np.sqrt((y * y).mean(-1)), 1.0, atol=1e-12)
    assert np.all(vae.rms_norm_c(np.zeros((1, 8)), g) == 0.0)   # the 1e-12 floor, no NaN


def test_nearest_upsample_closed_form():
    x = RNG.standard_normal((2, 3, 4, 2))
    y = vae.upsample_nearest2(x)
    assert y.shape == (2, 6, 8, 2)
    for h in range(6):
        for w in range(8):
            np.testing.assert_array_equal(y[:, h, w], x[:, h // 2, w // 2])


def test_temporal_upsample_frames():
    """Reading V5: T -> 1 + 2(T-1); frame 0 passes unchanged; output frames 2t-1, 2t are the two
    channel halves of the time-conv of input frame t; frame 0 never enters the time-conv."""
    C = 3
    x = RNG.standard_normal((4, 2, 2, C))
    w = RNG.standard_normal((2 * C, 3, 1, 1, C))
    b = RNG.standard_normal(2 * C)
    y = vae.temporal_upsample(x, w, b)
    assert y.shape[0] == 7
    np.testing.assert_array_equal(y[0], x[0])
    x2 = x.copy()
    x2[0] += 7.0                               # frame 0 is outside the time-conv history
    np.testing.assert_array_equal(vae.temporal_upsample(x2, w, b)[1:], y[1:])
    # frame 1 of the input sees zeros before it: its outputs are the last tap only
    last = np.einsum("hwc,oc->hwo", x[1], w[:, 2, 0, 0, :]) + b
    np.testing.assert_allclose(y[1], last[..., :C], atol=1e-12)
    np.testing.assert_allclose(y[2], last[..., C:], atol=1e-12)
    assert vae.temporal_upsample(x[:1], w, b).shape[0] == 1


def test_unpatchify_inverts_patchify():
    """Reading V6 against an independent patchify written as index loops."""
    F, Ht, Wt, C = 2, 3, 2, 16
    z = RNG.standard_normal((F, 2 * Ht, 2 * Wt, C))
    lat = np.zeros((F * Ht * Wt, 64))
    for f in range(F):
        for h in range(Ht):
            for w in range(Wt):
                for c in range(C):
                    for ph in range(2):
                        for pw in range(2):
                            lat[(f * Ht + h) * Wt + w, c * 4 + ph * 2 + pw] = z[f, 2 * h + ph, 2 * w + pw, c]
    np.testing.assert_array_equal(vae.unpatchify(lat, (F, Ht, Wt)), z)


def test_module_walk_matches_wan_widths():
    mods = sv.vae_modules(sv.WAN_VAE)
    convs = {n: (ci, co, k) for n, kind, ci, co, k in mods if kind == "conv"}
    assert convs["conv_in"] == (16, 384, (3, 3, 3))
    assert convs["up0.tconv"] == (384, 768, (3, 1, 1)) and convs["up0.sconv"] == (384, 192, (1, 3, 3))
    assert convs["up1.0.conv1"] == (192, 384, (3, 3, 3)) and convs["up1.0.skip"] == (192, 384, (1, 1, 1))
    assert convs["up2.0.conv1"] == (192, 192, (3, 3, 3)) and "up2.tconv" not in convs
    assert convs["up3.0.conv1"] == (96, 96, (3, 3, 3)) and convs["conv_out"] == (96, 3, (3, 3, 3))
    assert sv.output_frames(21) == 81 and sv.output_frames(1) == 1


@pytest.fixture(scope="module")
def tiny():
    shape = sv.TINY_VAE
    return shape, sv.vae_params(shape)


def test_decoder_shape_range_and_causality(tiny):
    """Output [1 + 4(F-1), 16 H_t, 16 W_t, 3] in [-1, 1]; frames decoded from latent frames < f do
    not change when later latent frames change (causal end to end)."""
    shape, params = tiny
    grid = (3, 2, 3)
    lat = RNG.standard_normal((np.prod(grid), 64))
    y = vae.decode(lat, grid, params, shape)
    assert y.shape == (9, 32, 48, 3)
    assert y.min() >= -1.0 and y.max() <= 1.0 and 0.0 < np.abs(y).mean() < 1.0
    lat2 = lat.copy()
    lat2[2 * 6:] += 3.0                         # latent frame 2 (rows of f = 2)
    y2 = vae.decode(lat2, grid, params, shape)
    np.testing.assert_array_equal(y[:5], y2[:5])     # output frames of latent frames 0, 1
    assert not np.allclose(y[5:], y2[5:])


def test_decoder_translation_equivariance_in_width(tiny):
    """Shifting the latent by one DiT token (2 latent pixels) along W shifts the interior of the
    video by 16 pixels: pins the upsampling index maps and the conv padding orientation."""
    shape, params = tiny
    F, Ht, Wt = 1, 1, 24
    z = RNG.standard_normal((F, Ht, Wt, 64))
    zs = np.zeros_like(z)
    zs[:, :, 1:] = z[:, :, :-1]
    y = vae.decode(z.reshape(-1, 64), (F, Ht, Wt), params, shape)
    ys = vae.decode(zs.reshape(-1, 64), (F, Ht, Wt), params, shape)
    # the receptive field (~16 latent pixels = 8 tokens each way) stays inside the grid for the
    # output columns of tokens 10..12
    np.testing.assert_allclose(ys[:, :, 16 * 11:16 * 14], y[:, :, 16 * 10:16 * 13], atol=1e-12)
    assert not np.allclose(ys[:, :, 16 * 10:16 * 13], y[:, :, 16 * 10:16 * 13])


def test_decode_flops_counts_every_conv(tiny, monkeypatch):
    """decode_flops (the bench's work count) equals 2 x MACs of the convolutions the decoder actually
    executes, recorded by wrapping causal_conv3d during a decode."""
    shape, params = tiny
    grid = (3, 2, 3)
    seen = []
    real = vae.causal_conv3d

    def rec(x, w, b):
        T, H, W, ci = x.shape
        co, kt, kh, kw, _ = w.shape
        seen.append(2 * T * H * W * co * ci * kt * kh * kw)
        return real(x, w, b)

    monkeypatch.setattr(vae, "causal_conv3d", rec)
    vae.decode(RNG.standard_normal((np.prod(grid), 64)), grid, params, shape)
    assert vae.decode_flops(grid, shape, sv.vae_modules) == sum(seen)
    assert len(seen) == sum(1 for m in sv.vae_modules(shape) if m[1] == "conv")
