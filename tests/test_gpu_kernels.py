"""Kernel parity on the GPU (rungs T1, T2): generator bitwise equality, tcgen05 GEMM with each
fused epilogue, tcgen05 flash attention (varlen, ragged tails, strided rows), time embedding —
each against the fp64 oracle on identical bf16 inputs, through the C-ABI."""
import numpy as np
import pytest

from oracle import dit
from synth import models as sm
from synth import rng
from tests.gpu_util import bf16_bits, from_dev_bf16, randn_bf16, rel_l2, to_dev, to_dev_bf16

pytestmark = pytest.mark.gpu

# Tolerances: a bf16-stored output carries RNE error <= 2^-9
# relative per element (rel-L2 <= 2^-9 ~ 1.95e-3); fp32 accumulation adds ~sqrt(K) 2^-24.
TOL_BF16_OUT = 3e-3
TOL_F32_OUT = 2e-5
TOL_ATTN = 6e-3   # P rounded to bf16 before PV (rel 2^-9) + O stored in bf16 (2^-9)


@pytest.fixture(scope="module")
def torch():
    import torch as t
    assert t.cuda.is_available()
    return t


@pytest.fixture(scope="module")
def ctx(torch):
    import paper_2604_04335_b200 as gs
    c = gs.Context(device=0)
    yield c
    c.close()


# ----------------------------------------------------------------------------- T1 generator
def test_weights_bitwise_equal_numpy_generator(ctx):
    shape = sm.ModelShape("t", 384, 6, 1536, 2, weight_seed=77)
    mid = ctx.model_create(shape.dim, shape.heads, shape.ffn, shape.layers, shape.weight_seed)
    for layer in range(shape.layers):
        ref = sm.block_params(shape, layer)
        for name, arr in ref.items():
            got = ctx.get_weight(mid, layer, name, arr.shape, arr.dtype)
            np.testing.assert_array_equal(got, arr, err_msg=f"layer {layer} {name}")
    for name, arr in sm.global_params(shape).items():
        got = ctx.get_weight(mid, -1, name, arr.shape, arr.dtype)
        np.testing.assert_array_equal(got, arr, err_msg=name)


def test_noise_bitwise_equal_numpy_generator(ctx):
    mid = ctx.model_create(384, 6, 1536, 1)
    req = ctx.submit(mid, 512, 256, 1, 50, 1003, [0])
    z = ctx.read_latent(req)
    np.testing.assert_array_equal(z, rng.noise_latent_f32(1003, 512))
    ctx.release(req)


# ----------------------------------------------------------------------------- T2 GEMM
GEMM_SHAPES = [(1, 64, 64), (127, 384, 384), (128, 1152, 384), (129, 256, 64), (300, 1536, 384),
               (1000, 64, 1536), (257, 4608, 1536)]


def _gemm_inputs(M, N, K, seed=0):
    g = np.random.default_rng(seed)
    a = randn_bf16(g, (M, K))
    w = bf16_bits(g.uniform(-1, 1, (N, K)) * np.sqrt(3.0 / K))
    b = bf16_bits(g.uniform(-0.1, 0.1, N))
    ref = dit.linear(rng.bf16_bits_to_f64(a), rng.bf16_bits_to_f64(w), rng.bf16_bits_to_f64(b))
    return a, w, b, ref


@pytest.mark.parametrize("M,N,K", GEMM_SHAPES)
def test_gemm_bf16_out(ctx, torch, M, N, K):
    import paper_2604_04335_b200 as gs
    a, w, b, ref = _gemm_inputs(M, N, K)
    out = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    ctx.debug_gemm(gs.EPI_BF16, M, N, K, to_dev_bf16(a), to_dev_bf16(w), to_dev_bf16(b), out)
    got = from_dev_bf16(out)
    assert rel_l2(got, ref) < TOL_BF16_OUT
    assert np.max(np.abs(got - ref) / (np.abs(ref) + 1e-2)) < 2 ** -7


@pytest.mark.parametrize("M,N,K", [(129, 1536, 384), (64, 256, 1536)])
def test_gemm_gelu(ctx, torch, M, N, K):
    import paper_2604_04335_b200 as gs
    a, w, b, ref = _gemm_inputs(M, N, K, seed=1)
    out = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    ctx.debug_gemm(gs.EPI_GELU_BF16, M, N, K, to_dev_bf16(a), to_dev_bf16(w), to_dev_bf16(b), out)
    assert rel_l2(from_dev_bf16(out), dit.gelu_tanh(ref)) < TOL_BF16_OUT


@pytest.mark.parametrize("M,N,K", [(200, 384, 64), (1000, 1536, 64)])
def test_gemm_f32(ctx, torch, M, N, K):
    import paper_2604_04335_b200 as gs
    a, w, b, ref = _gemm_inputs(M, N, K, seed=2)
    out = torch.empty((M, N), dtype=torch.float32, device="cuda")
    ctx.debug_gemm(gs.EPI_F32, M, N, K, to_dev_bf16(a), to_dev_bf16(w), to_dev_bf16(b), out)
    assert rel_l2(out.cpu().numpy(), ref) < TOL_F32_OUT


def test_gemm_gated_residual(ctx, torch):
    import paper_2604_04335_b200 as gs
    M, N, K, B = 333, 768, 1536, 3
    a, w, b, ref = _gemm_inputs(M, N, K, seed=3)
    g = np.random.default_rng(4)
    x0 = g.standard_normal((M, N)).astype(np.float32)
    ga = g.standard_normal(N).astype(np.float32)
    gb = g.standard_normal((B, 6 * N)).astype(np.float32)
    rows = np.sort(g.integers(0, B, M)).astype(np.int32)
    x = to_dev(x0, torch.float32)
    gbd = to_dev(gb, torch.float32)
    ctx.debug_gemm(gs.EPI_RESID_F32, M, N, K, to_dev_bf16(a), to_dev_bf16(w), to_dev_bf16(b), x,
                   gate_a=to_dev(ga, torch.float32), gate_b=gbd[:, 2 * N:], gate_b_stride=6 * N,
                   row_req=to_dev(rows, torch.int32))
    gate = ga[None, :].astype(np.float64) + gb[rows, 2 * N:3 * N]
    expect_delta = gate * ref
    assert rel_l2(x.cpu().numpy().astype(np.float64) - x0, expect_delta) < 1e-5


def test_gemm_euler(ctx, torch):
    import paper_2604_04335_b200 as gs
    M, N, K = 300, 64, 384
    a, w, b, ref = _gemm_inputs(M, N, K, seed=5)
    g = np.random.default_rng(6)
    z0 = g.standard_normal((M, N)).astype(np.float32)
    rows = np.r_[np.zeros(100), np.ones(200)].astype(np.int32)
    dsig = [-0.02, -0.05]
    z = to_dev(z0, torch.float32)
    ctx.debug_gemm(gs.EPI_EULER_F32, M, N, K, to_dev_bf16(a), to_dev_bf16(w), to_dev_bf16(b), z,
                   row_req=to_dev(rows, torch.int32), dsig=dsig)
    expect = np.array(dsig, np.float64)[rows][:, None] * ref
    assert rel_l2(z.cpu().numpy().astype(np.float64) - z0, expect) < 1e-5


def test_gemm_rows_bit_exact_across_M_and_position(ctx, torch):
    """A row's result must not depend on M or on its position inside a 128-row tile."""
    import paper_2604_04335_b200 as gs
    M, N, K = 700, 1536, 1536
    a, w, b, _ = _gemm_inputs(M, N, K, seed=7)
    A, W, Bv = to_dev_bf16(a), to_dev_bf16(w), to_dev_bf16(b)
    full = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    ctx.debug_gemm(gs.EPI_BF16, M, N, K, A, W, Bv, full)
    for lo, hi in [(0, 129), (5, 300), (77, 700), (699, 700)]:
        part = torch.empty((hi - lo, N), dtype=torch.bfloat16, device="cuda")
        ctx.debug_gemm(gs.EPI_BF16, hi - lo, N, K, A[lo:hi].contiguous(), W, Bv, part)
        assert torch.equal(part.view(torch.int16), full[lo:hi].view(torch.int16)), (lo, hi)


# ----------------------------------------------------------------------------- T2 attention
def _attn_case(seqlens, H, d, scale=1.0, seed=0):
    g = np.random.default_rng(seed)
    N = sum(seqlens)
    q, k, v = (randn_bf16(g, (N, H, d), scale if i < 2 else 1.0) for i in range(3))
    off = np.cumsum([0] + seqlens[:-1]).tolist()
    qf, kf, vf = (rng.bf16_bits_to_f64(x) for x in (q, k, v))
    ref = np.concatenate([dit.attention(qf[o:o + n], kf[o:o + n], vf[o:o + n])
                          for o, n in zip(off, seqlens)])
    return q, k, v, off, ref


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("seqlens", [[1], [127], [128], [129], [255, 256, 257], [300, 1, 513]])
def test_attention_varlen(ctx, torch, d, seqlens):
    H = 3
    q, k, v, off, ref = _attn_case(seqlens, H, d)
    o = torch.zeros((sum(seqlens), H, d), dtype=torch.bfloat16, device="cuda")
    ctx.debug_attention(to_dev_bf16(q), to_dev_bf16(k), to_dev_bf16(v), o, H, d, off, seqlens)
    assert rel_l2(from_dev_bf16(o), ref) < TOL_ATTN


@pytest.mark.parametrize("d", [64, 128])
def test_attention_sharp_logits_lazy_rescale(ctx, torch, d):
    # logit std ~ 16: the running max moves by > 2^8 often -> exercises the O rescale path
    seqlens = [1000]
    H = 2
    q, k, v, off, ref = _attn_case(seqlens, H, d, scale=4.0, seed=3)
    o = torch.zeros((1000, H, d), dtype=torch.bfloat16, device="cuda")
    ctx.debug_attention(to_dev_bf16(q), to_dev_bf16(k), to_dev_bf16(v), o, H, d, off, seqlens)
    assert rel_l2(from_dev_bf16(o), ref) < TOL_ATTN


def test_attention_strided_rows_and_batch_bit_exact(ctx, torch):
    """Q/K/V read from a [rows, 3, H, d] buffer (row stride 3Hd); a request gives identical
    bytes alone and packed with others (tiles start at request starts)."""
    H, d = 4, 128
    seqlens = [300, 700, 129]
    g = np.random.default_rng(9)
    N = sum(seqlens)
    qkv = randn_bf16(g, (N, 3, H, d))
    dev = to_dev_bf16(qkv)
    off = np.cumsum([0] + seqlens[:-1]).tolist()
    o = torch.zeros((N, H, d), dtype=torch.bfloat16, device="cuda")
    ctx.debug_attention(dev[:, 0], dev[:, 1], dev[:, 2], o, H, d, off, seqlens,
                        q_rs=3 * H * d, kv_rs=3 * H * d)
    f = rng.bf16_bits_to_f64(qkv)
    for o_, n in zip(off, seqlens):
        ref = dit.attention(f[o_:o_ + n, 0], f[o_:o_ + n, 1], f[o_:o_ + n, 2])
        assert rel_l2(from_dev_bf16(o[o_:o_ + n]), ref) < TOL_ATTN
    # request 1 alone
    alone = torch.zeros((700, H, d), dtype=torch.bfloat16, device="cuda")
    sub = dev[300:1000].contiguous()
    ctx.debug_attention(sub[:, 0], sub[:, 1], sub[:, 2], alone, H, d, [0], [700],
                        q_rs=3 * H * d, kv_rs=3 * H * d)
    assert torch.equal(alone.view(torch.int16), o[300:1000].view(torch.int16))


# ----------------------------------------------------------------------------- time embedding
def test_time_embedding(ctx):
    shape = sm.ModelShape("t", 384, 6, 1536, 1, weight_seed=5)
    mid = ctx.model_create(shape.dim, shape.heads, shape.ffn, shape.layers, shape.weight_seed)
    glob = sm.as_f64(sm.global_params(shape))
    ts = [1000.0, 993.5, 412.25, 0.0]
    e0, e = ctx.debug_time_embed(mid, ts, shape.dim)
    for i, t in enumerate(ts):
        r0, r = dit.time_embedding(np.float64(np.float32(t)), glob)
        assert rel_l2(e0[i], r0) < 1e-5
        assert rel_l2(e[i], r.reshape(-1)) < 1e-5


@pytest.mark.parametrize("epi", [0, 1, 3])
def test_gemm_pair_tile_width_does_not_change_bits(ctx, torch, epi):
    """The 192- and 256-wide pair tiles (the choice depends on the grid size, i.e. on M) give
    identical outputs, so SP degree / batch composition cannot change GEMM bits through it."""
    g = torch.Generator(device="cuda").manual_seed(5)
    M, N, K = 1000, 1536, 1536
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn(N, K, device="cuda", generator=g) * 0.03).to(torch.bfloat16)
    b = (torch.randn(N, device="cuda", generator=g) * 0.1).to(torch.bfloat16)
    ga = torch.rand(N, device="cuda", generator=g)
    gb = torch.rand(2, N, device="cuda", generator=g)
    rr = (torch.arange(M, device="cuda") % 2).to(torch.int32)
    outs = []
    for bn in (192, 256):
        ctx.set_option("gemm_bn", bn)
        if epi == 3:
            out = torch.randn(M, N, device="cuda", generator=torch.Generator(device="cuda").manual_seed(9))
            ctx.debug_gemm(epi, M, N, K, A, W, b, out, ga, gb, N, rr)
        else:
            out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
            ctx.debug_gemm(epi, M, N, K, A, W, b, out)
        outs.append(out.view(torch.int16 if out.dtype == torch.bfloat16 else torch.int32).cpu())
    ctx.set_option("gemm_bn", 0)
    assert torch.equal(outs[0], outs[1])


# ----------------------------------------------------------------------------- QKV epilogue sums of squares
@pytest.mark.parametrize("M,N,K,cols", [(300, 768, 256, 512), (1000, 15360 // 4, 1280, 2560)])
def test_gemm_ssq_partials(ctx, torch, M, N, K, cols):
    """per row and 32-column chunk the QKV GEMM epilogue writes sum (acc + bias)^2 in fp32 for
    the q | k columns.  Against the fp64 oracle linear on the same bf16 inputs (fp32 accumulation: ~1e-6 relative);
    chunks at or beyond ssq_cols are not written; the bf16 output equals the plain EPI_BF16 GEMM bit for bit."""
    import paper_2604_04335_b200 as gs
    a, w, b, ref = _gemm_inputs(M, N, K, seed=11)
    out = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    nc = cols // 32
    ssq = torch.full((M * nc + 64,), -7.0, dtype=torch.float32, device="cuda")  # sentinel tail
    ctx.debug_gemm_ssq(M, N, K, to_dev_bf16(a), to_dev_bf16(w), to_dev_bf16(b), out, ssq, cols)
    got = ssq.cpu().numpy()
    want = (ref[:, :cols] ** 2).reshape(M, nc, 32).sum(axis=2).reshape(-1)
    assert np.max(np.abs(got[:M * nc] - want) / want) < 1e-4
    assert np.all(got[M * nc:] == -7.0)
    plain = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    ctx.debug_gemm(gs.EPI_BF16, M, N, K, to_dev_bf16(a), to_dev_bf16(w), to_dev_bf16(b), plain)
    assert torch.equal(out.view(torch.int16), plain.view(torch.int16))


def test_gemm_ssq_bits_independent_of_M_and_tile_width(ctx, torch):
    """The partials of a row depend on that row alone: the same rows give the same bits inside a larger M and with
    the 192- or 256-wide pair tiles (chunks are 32-column aligned for both), so SP degree and batch composition
    cannot change the qk-RMSNorm through them."""
    g = torch.Generator(device="cuda").manual_seed(21)
    N, K, cols = 1536, 1536, 1024
    A = torch.randn(1000, K, device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn(N, K, device="cuda", generator=g) * 0.03).to(torch.bfloat16)
    b = (torch.randn(N, device="cuda", generator=g) * 0.1).to(torch.bfloat16)
    res = []
    for M, bn in ((1000, 256), (1000, 192), (333, 0)):
        ctx.set_option("gemm_bn", bn)
        out = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
        ssq = torch.empty((M * cols // 32,), dtype=torch.float32, device="cuda")
        ctx.debug_gemm_ssq(M, N, K, A[:M].contiguous(), W, b, out, ssq, cols)
        res.append(ssq.view(torch.int32).cpu().reshape(M, -1))
    ctx.set_option("gemm_bn", 0)
    assert torch.equal(res[0], res[1])
    assert torch.equal(res[0][:333], res[2])

