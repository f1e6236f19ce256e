"""Pins for the fp64 oracle (rung T0, SURVEY.md §4 / §8(c) pins P2-P5).

Each test fixes the oracle against something other than itself: brute force with
math.fsum loops, closed forms, invariants, special cases, or values the paper prints.
A plausible mistake (dropped term, wrong sign/index, transposed operand, swapped
modulation chunk) fails at least one of these.
"""
import math
import os

import numpy as np
import pytest

from oracle import dit
from synth import models as sm

RNG = np.random.default_rng(0)


# ----------------------------------------------------------------------------- attention (P2)
def _attention_bruteforce(q, k, v):
    n_q, H, d = q.shape
    n = k.shape[0]
    out = np.zeros((n_q, H, d))
    for h in range(H):
        for i in range(n_q):
            logits = [math.fsum(q[i, h, c] * k[j, h, c] for c in range(d)) / math.sqrt(d)
                      for j in range(n)]
            m = max(logits)
            w = [math.exp(s - m) for s in logits]
            z = math.fsum(w)
            for c in range(d):
                out[i, h, c] = math.fsum(w[j] * v[j, h, c] for j in range(n)) / z
    return out


@pytest.mark.parametrize("n,H,d", [(1, 1, 2), (5, 2, 4), (8, 3, 8), (7, 1, 6)])
def test_attention_bruteforce(n, H, d):
    q, k, v = (RNG.standard_normal((n, H, d)) * 2 for _ in range(3))
    np.testing.assert_allclose(dit.attention(q, k, v), _attention_bruteforce(q, k, v),
                               rtol=0, atol=1e-13)


def test_attention_q_zero_is_mean_v():
    k, v = RNG.standard_normal((2, 9, 3, 8))
    q = np.zeros((9, 3, 8))
    np.testing.assert_allclose(dit.attention(q, k, v), np.broadcast_to(v.mean(0), v.shape),
                               atol=1e-14)


def test_attention_one_token_returns_v():
    q, k, v = RNG.standard_normal((3, 1, 4, 16))
    np.testing.assert_allclose(dit.attention(q, k, v), v, atol=1e-15)


def test_attention_logit_row_shift_invariance():
    # K <- K + 1 c^T adds q_i.c to every logit of row i: softmax unchanged
    q, k, v = RNG.standard_normal((3, 6, 2, 8))
    c = RNG.standard_normal((1, 2, 8))
    np.testing.assert_allclose(dit.attention(q, k + c, v), dit.attention(q, k, v), atol=1e-12)


def test_softmax_rows_sum_to_one():
    s = RNG.standard_normal((4, 7)) * 30
    np.testing.assert_allclose(dit.softmax(s).sum(-1), 1.0, atol=1e-15)


def test_attention_is_not_transposed():
    # non-symmetric check: output row i must be a convex combination of V rows with
    # weights from q_i (swap q/k would break this for a single query)
    q = np.array([[[10.0, 0.0]]])
    k = np.array([[[1.0, 0.0]], [[-1.0, 0.0]]])
    v = np.array([[[1.0, 2.0]], [[3.0, 4.0]]])
    o = dit.attention(q, k, v)[0, 0]
    w1 = 1.0 / (1.0 + math.exp(-20.0 / math.sqrt(2)))
    np.testing.assert_allclose(o, w1 * v[0, 0] + (1 - w1) * v[1, 0], atol=1e-14)


# ----------------------------------------------------------------------------- components (P4)
def test_layer_norm_constant_row_is_zero():
    x = np.full((3, 16), 2.5)
    assert np.all(dit.layer_norm(x) == 0.0)


def test_layer_norm_closed_form():
    x = np.array([[1.0, 2.0, 3.0, 4.0]])
    var = 1.25  # biased variance of 1..4
    np.testing.assert_allclose(dit.layer_norm(x, eps=0.0),
                               (x - 2.5) / math.sqrt(var), atol=1e-15)


def test_rms_norm_constant_vector():
    c, D = 0.3, 12
    g = RNG.standard_normal(D)
    np.testing.assert_allclose(dit.rms_norm(np.full((1, D), c), g),
                               (c / math.sqrt(c * c + 1e-6)) * g[None], atol=1e-15)


def test_gelu_tanh_values():
    np.testing.assert_allclose(dit.gelu_tanh(np.array([0.0, 1.0, -1.0])),
                               [0.0, 0.841192, -0.158808], atol=5e-7)


def test_modulate_closed_form():
    a = np.array([2.0]); sh = np.array([0.5]); sc = np.array([-0.25])
    assert dit.modulate(a, sh, sc)[0] == 2.0 * 0.75 + 0.5


def test_rope_slots_closed_form():
    assert dit.rope_slots(128) == (22, 21, 21)
    assert dit.rope_slots(64) == (12, 10, 10)
    for d in (64, 96, 128):
        assert sum(dit.rope_slots(d)) == d // 2


def test_rope_identity_at_origin_and_norm_preserving():
    d, H = 64, 3
    x = RNG.standard_normal((5, H, d))
    pos0 = np.zeros((5, 3), dtype=int)
    np.testing.assert_array_equal(dit.rope_apply(x, dit.rope_angles(pos0, d)), x)
    pos = RNG.integers(0, 50, size=(5, 3))
    y = dit.rope_apply(x, dit.rope_angles(pos, d))
    np.testing.assert_allclose(np.linalg.norm(y, axis=-1), np.linalg.norm(x, axis=-1), rtol=1e-13)


def test_rope_matches_complex_multiply():
    d = 128
    x = RNG.standard_normal((4, 2, d))
    pos = np.array([[0, 0, 0], [1, 2, 3], [20, 44, 79], [5, 0, 7]])
    # independent formulation: complex numbers, per-axis frequency table written out
    slots = [22, 21, 21]
    freqs = []
    for a, s in enumerate(slots):
        for j in range(s):
            freqs.append((a, 10000.0 ** (-(2.0 * j) / (2 * s))))
    xc = x[..., 0::2] + 1j * x[..., 1::2]
    rot = np.array([[np.exp(1j * p[a] * f) for (a, f) in freqs] for p in pos])
    yc = xc * rot[:, None, :]
    y = dit.rope_apply(x, dit.rope_angles(pos, d))
    np.testing.assert_allclose(y[..., 0::2], yc.real, atol=1e-12)
    np.testing.assert_allclose(y[..., 1::2], yc.imag, atol=1e-12)


def test_rope_relative_position():
    d = 64
    q, k = RNG.standard_normal((2, 1, 1, d))
    m, n = np.array([[3, 5, 7]]), np.array([[1, 9, 2]])
    delta = np.array([[4, 11, 6]])

    def dot(a, b):
        qa = dit.rope_apply(q, dit.rope_angles(a, d))
        kb = dit.rope_apply(k, dit.rope_angles(b, d))
        return float((qa * kb).sum())
    assert abs(dot(m, n) - dot(m + delta, n + delta)) < 1e-12
    assert abs(dot(m, n) - dot(m + delta, n)) > 1e-6


def test_token_positions_row_order():
    pos = dit.token_positions((2, 3, 4))
    assert pos.shape == (24, 3)
    assert tuple(pos[0]) == (0, 0, 0) and tuple(pos[1]) == (0, 0, 1)
    assert tuple(pos[4]) == (0, 1, 0) and tuple(pos[12]) == (1, 0, 0)
    assert tuple(pos[23]) == (1, 2, 3)


def test_linear_against_fsum_loop():
    x = RNG.standard_normal((3, 7)); w = RNG.standard_normal((5, 7)); b = RNG.standard_normal(5)
    ref = np.array([[math.fsum(x[i, c] * w[j, c] for c in range(7)) + b[j] for j in range(5)]
                    for i in range(3)])
    np.testing.assert_allclose(dit.linear(x, w, b), ref, atol=1e-14)


# ----------------------------------------------------------------------------- block (P3)
def _tiny_block(D=48, H=4, F=96, seed=3):
    shape = sm.ModelShape("t", D, H, F, 1, weight_seed=seed)
    return shape, sm.as_f64(sm.block_params(shape, 0))


def _reqs(ns_grids):
    off, out = 0, []
    for g in ns_grids:
        n = g[0] * g[1] * g[2]
        out.append((off, n, g))
        off += n
    return out, off


def test_block_zero_gates_is_identity():
    shape, blk = _tiny_block()
    blk["mod"][2] = 0.0
    blk["mod"][5] = 0.0
    reqs, N = _reqs([(1, 3, 4)])
    x = RNG.standard_normal((N, shape.dim))
    e = RNG.standard_normal((1, 6, shape.dim))
    e[:, 2] = 0.0
    e[:, 5] = 0.0
    np.testing.assert_array_equal(dit.dit_block(x, blk, e, reqs, shape.heads), x)


def test_block_attention_branch_closed_form():
    # sc1 = -1, sh1 = 0  =>  a = 0  =>  v = b_v for every token  =>  O = b_v (softmax sums
    # to one)  =>  with g2 = 0: x_out = x + g1 * (b_v W_o^T + b_o), independent of x.
    shape, blk = _tiny_block()
    D = shape.dim
    blk["mod"][:] = 0.0
    e = np.zeros((1, 6, D))
    e[0, 1] = -1.0                      # sc1
    g1 = RNG.standard_normal(D)
    e[0, 2] = g1                        # g1
    reqs, N = _reqs([(2, 2, 3)])
    x = RNG.standard_normal((N, D))
    b_v = blk["b_qkv"][2 * D:]
    expect = x + g1 * (b_v @ blk["w_o"].T + blk["b_o"])
    np.testing.assert_allclose(dit.dit_block(x, blk, e, reqs, shape.heads), expect, atol=1e-12)


def test_block_mlp_branch_closed_form():
    # g1 = 0, sc2 = -1, sh2 = c  =>  x_out = x + g2 * (GELU(c W_1^T + b_1) W_2^T + b_2)
    shape, blk = _tiny_block()
    D = shape.dim
    blk["mod"][:] = 0.0
    e = np.zeros((1, 6, D))
    c = RNG.standard_normal(D)
    g2 = RNG.standard_normal(D)
    e[0, 3], e[0, 4], e[0, 5] = c, -1.0, g2
    reqs, N = _reqs([(1, 4, 2)])
    x = RNG.standard_normal((N, D))
    mlp = dit.gelu_tanh(c @ blk["w_1"].T + blk["b_1"]) @ blk["w_2"].T + blk["b_2"]
    np.testing.assert_allclose(dit.dit_block(x, blk, e, reqs, shape.heads), x + g2 * mlp,
                               atol=1e-12)


def test_block_q_zero_attention_is_mean_of_v():
    # W_q = b_q = 0 => q = 0 after RMSNorm/RoPE => O = per-request mean of v
    shape, blk = _tiny_block()
    D, H = shape.dim, shape.heads
    blk["w_qkv"][:D] = 0.0
    blk["b_qkv"][:D] = 0.0
    blk["mod"][:] = 0.0
    e = np.zeros((2, 6, D))
    e[:, 2] = 1.0                       # g1 = 1, g2 = 0
    reqs, N = _reqs([(1, 2, 3), (1, 1, 5)])
    x = RNG.standard_normal((N, D))
    out = dit.dit_block(x, blk, e, reqs, H)
    a = dit.layer_norm(x)
    v = a @ blk["w_qkv"][2 * D:].T + blk["b_qkv"][2 * D:]
    for off, n, _g in reqs:
        o = v[off:off + n].mean(0)
        expect = x[off:off + n] + (o @ blk["w_o"].T + blk["b_o"])
        np.testing.assert_allclose(out[off:off + n], expect, atol=1e-12)


def test_block_permutation_equivariance():
    shape, blk = _tiny_block()
    D = shape.dim
    grid = (2, 3, 4)
    n = 24
    x = RNG.standard_normal((n, D))
    e = RNG.standard_normal((1, 6, D)) * 0.3
    pos = dit.token_positions(grid)
    perm = RNG.permutation(n)
    y = dit.dit_block(x, blk, e, [(0, n, pos)], shape.heads)
    yp = dit.dit_block(x[perm], blk, e, [(0, n, pos[perm])], shape.heads)
    np.testing.assert_allclose(yp, y[perm], atol=1e-12)


def test_block_varlen_packing_equals_alone():
    shape, blk = _tiny_block()
    D = shape.dim
    grids = [(1, 2, 3), (2, 2, 2), (1, 1, 1)]
    reqs, N = _reqs(grids)
    x = RNG.standard_normal((N, D))
    e = RNG.standard_normal((3, 6, D)) * 0.3
    packed = dit.dit_block(x, blk, e, reqs, shape.heads)
    for r, (off, n, g) in enumerate(reqs):
        alone = dit.dit_block(x[off:off + n], blk, e[r:r + 1], [(0, n, g)], shape.heads)
        np.testing.assert_allclose(packed[off:off + n], alone, atol=1e-13)


def test_steps_varlen_packing_equals_alone():
    """A batch's step == each request stepped alone (different step indices; the basis of
    tests/gpu_util.oracle_steps_per_request)."""
    shape = sm.TINY.with_layers(2)
    glob = sm.as_f64(sm.global_params(shape))
    blocks = [sm.as_f64(sm.block_params(shape, l)) for l in range(shape.layers)]
    grids = [(1, 2, 3), (2, 2, 2)]
    zs = [RNG.standard_normal((int(np.prod(g)), shape.lat)) for g in grids]
    packed = dit.dit_steps(zs, grids, [0, 7], 50, 2, glob, blocks, shape.heads)
    for z, g, i, p in zip(zs, grids, [0, 7], packed):
        alone = dit.dit_steps([z], [g], [i], 50, 2, glob, blocks, shape.heads)[0]
        np.testing.assert_allclose(p, alone, rtol=0, atol=1e-12 * np.abs(alone).max())


def test_block_rows_sampled_equals_full():
    shape, blk = _tiny_block()
    grid = (2, 3, 5)
    n = 30
    x = RNG.standard_normal((n, shape.dim))
    e = RNG.standard_normal((6, shape.dim)) * 0.3
    full = dit.dit_block(x, blk, e[None], [(0, n, grid)], shape.heads)
    rows = [0, 7, 13, 29]
    np.testing.assert_allclose(dit.dit_block_rows(x, blk, e, grid, shape.heads, rows),
                               full[rows], atol=1e-12)


# ----------------------------------------------------------------------------- step (P5)
def _golden_sigmas():
    path = os.path.join(os.path.dirname(__file__), "golden", "sigma_schedule.txt")
    return [tuple(map(float, l.split())) for l in open(path) if l.strip() and l[0] != "#"]


def test_sigma_schedule_golden():
    sig = dit.sigmas(50, 5.0)
    assert sig[0] == 1.0 and sig[-1] == 0.0
    assert np.all(np.diff(sig) < 0)
    for i, s in _golden_sigmas():
        assert abs(sig[int(i)] - s) < 1e-15


def test_sigma_shift_one_is_linear():
    np.testing.assert_allclose(dit.sigmas(10, 1.0), 1 - np.arange(11) / 10, atol=1e-15)


def test_sinusoid_at_zero():
    s = dit.sinusoid(0.0)
    np.testing.assert_array_equal(s, np.r_[np.ones(128), np.zeros(128)])


def test_sinusoid_frequencies():
    s = dit.sinusoid(1.0)
    assert abs(s[0] - math.cos(1.0)) < 1e-15 and abs(s[128] - math.sin(1.0)) < 1e-15
    w = 10000.0 ** (-64 / 128)
    assert abs(s[64] - math.cos(w)) < 1e-15 and abs(s[192] - math.sin(w)) < 1e-15


def test_time_embedding_closed_form():
    shape = sm.ModelShape("t", 16, 2, 32, 1)
    g = sm.as_f64(sm.global_params(shape))
    g["w_t1"][:] = 0.0
    g["b_t1"][:] = 0.0
    e0, e = dit.time_embedding(123.0, g)
    np.testing.assert_array_equal(e0, g["b_t2"])
    silu = g["b_t2"] / (1 + np.exp(-g["b_t2"]))
    np.testing.assert_allclose(e.reshape(-1), g["w_tp"] @ silu + g["b_tp"], atol=1e-14)


def test_euler_closed_forms():
    z = RNG.standard_normal((4, 64)); v = RNG.standard_normal((4, 64))
    np.testing.assert_array_equal(dit.euler(z, 0 * v, 0.9, 0.8), z)
    d1 = dit.euler(z, v, 0.9, 0.8) - z
    d2 = dit.euler(z, 2 * v, 0.9, 0.8) - z
    np.testing.assert_allclose(d2, 2 * d1, atol=1e-15)
    np.testing.assert_allclose(d1, -0.1 * v, atol=1e-15)


def test_steps_k0_identity_and_k_composes():
    shape = sm.ModelShape("t", 24, 2, 48, 2)
    glob = sm.as_f64(sm.global_params(shape))
    blocks = [sm.as_f64(sm.block_params(shape, l)) for l in range(2)]
    z = [RNG.standard_normal((6, 64)), RNG.standard_normal((4, 64))]
    grids = [(1, 2, 3), (1, 2, 2)]
    out0 = dit.dit_steps(z, grids, [0, 5], 10, 0, glob, blocks, shape.heads)
    for a, b in zip(out0, z):
        np.testing.assert_array_equal(a, b)
    two = dit.dit_steps(z, grids, [0, 5], 10, 2, glob, blocks, shape.heads)
    one = dit.dit_steps(z, grids, [0, 5], 10, 1, glob, blocks, shape.heads)
    oneone = dit.dit_steps(one, grids, [1, 6], 10, 1, glob, blocks, shape.heads)
    for a, b in zip(two, oneone):
        np.testing.assert_array_equal(a, b)


def test_head_closed_form():
    # constant rows => LN = 0 => v = hsh W_head^T + b_head with hsh = M_head[0] + e0
    shape = sm.ModelShape("t", 16, 2, 32, 1)
    g = sm.as_f64(sm.global_params(shape))
    x = np.full((3, 16), 1.7)
    e0 = RNG.standard_normal(16)
    v = dit.head(x, np.broadcast_to(e0, (3, 16)), g)
    np.testing.assert_allclose(v, np.broadcast_to((g["mod_head"][0] + e0) @ g["w_head"].T
                                                  + g["b_head"], (3, 64)), atol=1e-13)


# ----------------------------------------------------------------------------- NEXT-1: text cross-attention + CFG
def _text_shape(D=48, H=3, L=5, T=16):
    return sm.ModelShape("tx", D, H, 2 * D, 1, weight_seed=91).with_text(L, T)


def _fsum_linear(x, w, b):
    return np.array([[math.fsum(x[i, k] * w[o, k] for k in range(x.shape[1])) + b[o]
                      for o in range(w.shape[0])] for i in range(x.shape[0])])


def test_text_embedding_against_fsum():
    shape = _text_shape()
    glob = sm.as_f64(sm.global_params(shape))
    emb = RNG.standard_normal((shape.text_len, shape.text_dim))
    h = _fsum_linear(emb, glob["w_te1"], glob["b_te1"])
    h = 0.5 * h * (1 + np.tanh(math.sqrt(2 / math.pi) * (h + 0.044715 * h ** 3)))
    ref = _fsum_linear(h, glob["w_te2"], glob["b_te2"])
    np.testing.assert_allclose(dit.text_embedding(emb, glob), ref, rtol=1e-12, atol=1e-12)


def test_layer_norm_affine_constant_row_is_beta():
    w, b = RNG.standard_normal(8), RNG.standard_normal(8)
    np.testing.assert_allclose(dit.layer_norm_affine(np.full((2, 8), 3.25), w, b), np.tile(b, (2, 1)),
                               atol=1e-12)


def test_cross_attention_zero_query_is_mean_of_context_values():
    """W_cq = b_cq = 0 -> q = 0 -> uniform weights over the L context tokens: every row gets
    mean_L(c W_cv^T + b_cv) W_co^T + b_co."""
    shape = _text_shape()
    blk = sm.as_f64(sm.block_params(shape, 0))
    blk["w_cq"][:] = 0
    blk["b_cq"][:] = 0
    D = shape.dim
    x = RNG.standard_normal((7, D))
    c = RNG.standard_normal((shape.text_len, D))
    v = c @ blk["w_ckv"][D:].T + blk["b_ckv"][D:]
    want = v.mean(axis=0) @ blk["w_co"].T + blk["b_co"]
    np.testing.assert_allclose(dit.cross_attention(x, blk, c, shape.heads), np.tile(want, (7, 1)),
                               rtol=1e-10, atol=1e-10)


def test_cross_attention_single_context_token_returns_its_value():
    shape = _text_shape(L=1)
    blk = sm.as_f64(sm.block_params(shape, 0))
    D = shape.dim
    x = RNG.standard_normal((4, D))
    c = RNG.standard_normal((1, D))
    want = (c @ blk["w_ckv"][D:].T + blk["b_ckv"][D:]) @ blk["w_co"].T + blk["b_co"]
    np.testing.assert_allclose(dit.cross_attention(x, blk, c, shape.heads), np.tile(want, (4, 1)),
                               rtol=1e-10, atol=1e-10)


def test_cross_attention_context_permutation_invariant_and_row_wise():
    shape = _text_shape(L=6)
    blk = sm.as_f64(sm.block_params(shape, 0))
    x = RNG.standard_normal((5, shape.dim))
    c = RNG.standard_normal((6, shape.dim))
    out = dit.cross_attention(x, blk, c, shape.heads)
    perm = RNG.permutation(6)
    np.testing.assert_allclose(dit.cross_attention(x, blk, c[perm], shape.heads), out, rtol=1e-11,
                               atol=1e-12)
    np.testing.assert_allclose(dit.cross_attention(x[2:4], blk, c, shape.heads), out[2:4], rtol=1e-12,
                               atol=1e-13)


def test_cross_attention_against_bruteforce_heads():
    shape = _text_shape(D=12, H=2, L=4)
    blk = sm.as_f64(sm.block_params(shape, 0))
    D, H, d = 12, 2, 6
    x = RNG.standard_normal((3, D))
    c = RNG.standard_normal((4, D))
    a = (x - x.mean(1, keepdims=True)) / np.sqrt(x.var(1, keepdims=True) + 1e-6) * blk["ln3_w"] + blk["ln3_b"]
    q = _fsum_linear(a, blk["w_cq"], blk["b_cq"])
    q = q / np.sqrt((q * q).mean(1, keepdims=True) + 1e-6) * blk["g_cq"]
    kv = _fsum_linear(c, blk["w_ckv"], blk["b_ckv"])
    k = kv[:, :D] / np.sqrt((kv[:, :D] ** 2).mean(1, keepdims=True) + 1e-6) * blk["g_ck"]
    o = _attention_bruteforce(q.reshape(3, H, d), k.reshape(4, H, d), kv[:, D:].reshape(4, H, d))
    ref = _fsum_linear(o.reshape(3, D), blk["w_co"], blk["b_co"])
    np.testing.assert_allclose(dit.cross_attention(x, blk, c, H), ref, rtol=1e-10, atol=1e-12)


def test_block_with_cross_attention_reduces_to_self_block_when_w_co_zero():
    shape = _text_shape()
    blk = sm.as_f64(sm.block_params(shape, 0))
    blk["w_co"][:] = 0
    blk["b_co"][:] = 0
    grid = (1, 2, 3)
    x = RNG.standard_normal((6, shape.dim))
    e = RNG.standard_normal((1, 6, shape.dim)) * 0.1
    c = RNG.standard_normal((shape.text_len, shape.dim))
    a = dit.dit_block(x, blk, e, [(0, 6, grid)], shape.heads, [c])
    b = dit.dit_block(x, blk, e, [(0, 6, grid)], shape.heads)
    np.testing.assert_array_equal(a, b)


def test_cfg_closed_forms():
    vc, vu = RNG.standard_normal((5, 4)), RNG.standard_normal((5, 4))
    np.testing.assert_allclose(dit.cfg_velocity(vc, vu, 1.0), vc, rtol=0, atol=1e-15)
    np.testing.assert_array_equal(dit.cfg_velocity(vc, vu, 0.0), vu)
    np.testing.assert_allclose(dit.cfg_velocity(vc, vu, 2.5) - dit.cfg_velocity(vc, vu, 1.5), vc - vu,
                               atol=1e-12)


def test_steps_with_cfg_scale_one_equals_cond_only():
    shape = sm.TINY.with_layers(1).with_text(8, 32)
    glob = sm.as_f64(sm.global_params(shape))
    blocks = [sm.as_f64(sm.block_params(shape, 0))]
    z = RNG.standard_normal((12, 64))
    pc = sm.as_f64({"p": sm.prompt_embeds(shape, 4, 0)})["p"]
    pu = sm.as_f64({"p": sm.prompt_embeds(shape, 4, 1)})["p"]
    a = dit.dit_steps([z], [(1, 3, 4)], [3], 50, 1, glob, blocks, shape.heads, prompts=[(pc, pu)],
                      cfg=[1.0])[0]
    b = dit.dit_steps([z], [(1, 3, 4)], [3], 50, 1, glob, blocks, shape.heads, prompts=[(pc, None)])[0]
    np.testing.assert_allclose(a, b, rtol=0, atol=1e-12)
    c = dit.dit_steps([z], [(1, 3, 4)], [3], 50, 1, glob, blocks, shape.heads, prompts=[(pu, None)])[0]
    g0 = dit.dit_steps([z], [(1, 3, 4)], [3], 50, 1, glob, blocks, shape.heads, prompts=[(pc, pu)],
                       cfg=[0.0])[0]
    np.testing.assert_allclose(g0, c, rtol=0, atol=1e-12)


# ----------------------------------------------------------------------------- whole-block / time-MLP brute force
# Scalar math.fsum re-statements of SURVEY.md §8(c) "Block" steps 1-7 and "Step" (time MLP),
# written from the text, not from oracle/dit.py: they pin the q/k branch (RMSNorm over the FULL
# D, the gains g_q / g_k applied before RoPE, the per-axis RoPE slot split and frequencies, the
# request-local (f, h, w) positions) and the time MLP's first Linear + SiLU.
def _fs_ln(row):
    mu = math.fsum(row) / len(row)
    var = math.fsum((t - mu) ** 2 for t in row) / len(row)
    return [(t - mu) / math.sqrt(var + 1e-6) for t in row]


def _fs_lin(row, w, b):
    return [math.fsum(row[c] * w[o][c] for c in range(len(row))) + b[o] for o in range(len(w))]


def _fs_rope(vec, pos, d):
    """Consecutive pairs (2j, 2j+1) rotated by theta = pos_a * 10000^(-2j'/m_a); slots
    [d/2 - 2 floor(d/6), floor(d/6), floor(d/6)] for axes (f, h, w), j' the slot within its axis,
    m_a = 2 * slots_a (SURVEY.md §8(c) Block step 4)."""
    s = d // 6
    slots = [d // 2 - 2 * s, s, s]
    out, pair = list(vec), 0
    for a in range(3):
        for jj in range(slots[a]):
            th = pos[a] * 10000.0 ** (-2.0 * jj / (2 * slots[a]))
            x0, x1 = vec[2 * pair], vec[2 * pair + 1]
            out[2 * pair] = x0 * math.cos(th) - x1 * math.sin(th)
            out[2 * pair + 1] = x0 * math.sin(th) + x1 * math.cos(th)
            pair += 1
    return out


def _fs_gelu(u):
    return 0.5 * u * (1.0 + math.tanh(math.sqrt(2.0 / math.pi) * (u + 0.044715 * u ** 3)))


def _fs_block(x, blk, e_req, reqs, H):
    N, D = len(x), len(x[0])
    d = D // H
    w_qkv, b_qkv = blk["w_qkv"].tolist(), blk["b_qkv"].tolist()
    gq, gk = blk["g_q"].tolist(), blk["g_k"].tolist()
    out = [None] * N
    for r, (off, n, grid) in enumerate(reqs):
        F_, Ht, Wt = grid
        mod = [[blk["mod"][c][i] + e_req[r][c][i] for i in range(D)] for c in range(6)]
        sh1, sc1, g1, sh2, sc2, g2 = mod
        q, k, v = [], [], []
        for t in range(n):
            a = [ln * (1 + sc1[i]) + sh1[i] for i, ln in enumerate(_fs_ln(x[off + t]))]
            y = _fs_lin(a, w_qkv, b_qkv)
            pos = (t // (Ht * Wt), (t // Wt) % Ht, t % Wt)   # request-local index -> (f, h, w)
            qr, kr = y[:D], y[D:2 * D]
            rq = math.sqrt(math.fsum(c * c for c in qr) / D + 1e-6)   # RMS over the full D
            rk = math.sqrt(math.fsum(c * c for c in kr) / D + 1e-6)
            qn = [qr[i] / rq * gq[i] for i in range(D)]
            kn = [kr[i] / rk * gk[i] for i in range(D)]
            q.append([_fs_rope(qn[h * d:(h + 1) * d], pos, d) for h in range(H)])
            k.append([_fs_rope(kn[h * d:(h + 1) * d], pos, d) for h in range(H)])
            v.append([y[2 * D + h * d:2 * D + (h + 1) * d] for h in range(H)])
        for t in range(n):
            o = []
            for h in range(H):
                lg = [math.fsum(q[t][h][c] * k[u][h][c] for c in range(d)) / math.sqrt(d) for u in range(n)]
                m = max(lg)
                p = [math.exp(s - m) for s in lg]
                z = math.fsum(p)
                o += [math.fsum(p[u] * v[u][h][c] for u in range(n)) / z for c in range(d)]
            ao = _fs_lin(o, blk["w_o"].tolist(), blk["b_o"].tolist())
            x1 = [x[off + t][i] + g1[i] * ao[i] for i in range(D)]
            a2 = [ln * (1 + sc2[i]) + sh2[i] for i, ln in enumerate(_fs_ln(x1))]
            hdn = [_fs_gelu(u) for u in _fs_lin(a2, blk["w_1"].tolist(), blk["b_1"].tolist())]
            mo = _fs_lin(hdn, blk["w_2"].tolist(), blk["b_2"].tolist())
            out[off + t] = [x1[i] + g2[i] * mo[i] for i in range(D)]
    return np.array(out)


def test_block_against_fsum_bruteforce_with_rope_and_gains():
    """Whole tiny block (D = 24, H = 2, d = 12: RoPE slots (2, 2, 2), frequencies 1 and 1/100)
    over two requests with non-trivial positions on every axis, strongly non-uniform gains and
    per-request modulation: catches RMSNorm per head instead of over D, gains after RoPE or
    dropped, a wrong slot split / frequency / position, batch-global instead of request-local
    positions, and a swapped modulation chunk."""
    D, H = 24, 2
    shape = sm.ModelShape("bf", D, H, 40, 1, weight_seed=17)
    blk = sm.as_f64(sm.block_params(shape, 0))
    g = np.random.default_rng(5)
    blk["g_q"] = 1.0 + g.standard_normal(D)          # gains far from 1: order / scope visible
    blk["g_k"] = 1.0 + g.standard_normal(D)
    blk["w_qkv"][:2 * D] *= 3.0                       # sharper logits: RoPE errors move the softmax
    grids = [(2, 2, 3), (1, 2, 2)]
    reqs, N = _reqs(grids)
    x = g.standard_normal((N, D)) * 1.5 + 0.3
    e = g.standard_normal((2, 6, D)) * 0.4
    ref = _fs_block(x.tolist(), blk, e.tolist(), reqs, H)
    np.testing.assert_allclose(dit.dit_block(x, blk, e, reqs, H), ref, rtol=0, atol=1e-12)


def test_time_embedding_against_fsum_bruteforce():
    """e0 = W_t2 SiLU(W_t1 s(t) + b_t1) + b_t2, e = W_tp SiLU(e0) + b_tp with every weight
    non-zero (SURVEY.md §8(c) "Step"): pins the first Linear and both SiLUs."""
    shape = sm.ModelShape("t", 16, 2, 32, 1, weight_seed=23)
    gl = sm.as_f64(sm.global_params(shape))
    t = 731.25
    half = 128
    s = [math.cos(t * 10000.0 ** (-j / half)) for j in range(half)] + \
        [math.sin(t * 10000.0 ** (-j / half)) for j in range(half)]
    silu = lambda u: u / (1.0 + math.exp(-u))   # noqa: E731
    h1 = [silu(u) for u in _fs_lin(s, gl["w_t1"].tolist(), gl["b_t1"].tolist())]
    e0 = _fs_lin(h1, gl["w_t2"].tolist(), gl["b_t2"].tolist())
    e = _fs_lin([silu(u) for u in e0], gl["w_tp"].tolist(), gl["b_tp"].tolist())
    got_e0, got_e = dit.time_embedding(t, gl)
    np.testing.assert_allclose(got_e0, e0, rtol=0, atol=1e-12)
    np.testing.assert_allclose(got_e.reshape(-1), e, rtol=0, atol=1e-12)
    # the first SiLU matters: dropping it changes e0 by far more than the tolerance
    no_silu = _fs_lin(_fs_lin(s, gl["w_t1"].tolist(), gl["b_t1"].tolist()), gl["w_t2"].tolist(),
                      gl["b_t2"].tolist())
    assert np.max(np.abs(np.array(no_silu) - got_e0)) > 1e-3
