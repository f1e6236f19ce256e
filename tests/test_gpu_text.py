"""Text cross-attention + classifier-free guidance on the GPU: generator
bitwise equality for the new tensors and prompts, block / step parity against the fp64 oracle, and
bit-exactness across SP degree, batch composition and preempt -> re-shard -> resume."""
import numpy as np
import pytest

from oracle import dit
from synth import models as sm
from synth import rng
from tests.gpu_util import rel_l2

pytestmark = pytest.mark.gpu

TOL = 1e-2
TINY_T = sm.TINY.with_layers(2).with_text(64, 256)


@pytest.fixture(scope="module")
def gs():
    import paper_2604_04335_b200 as m
    m.load()
    return m


def _mk(ctx, shape, layers=None):
    return ctx.model_create(shape.dim, shape.heads, shape.ffn, layers or shape.layers, shape.weight_seed,
                            cross_attn=True, text_len=shape.text_len, text_dim=shape.text_dim)


def test_text_weights_bitwise_equal_numpy_generator(gs):
    ctx = gs.Context(device=0)
    mid = _mk(ctx, TINY_T)
    for name in ("ln3_w", "ln3_b", "w_cq", "b_cq", "w_ckv", "b_ckv", "g_cq", "g_ck", "w_co", "b_co"):
        ref = sm.block_params(TINY_T, 1)[name]
        np.testing.assert_array_equal(ctx.get_weight(mid, 1, name, ref.shape, ref.dtype), ref, err_msg=name)
    for name in ("w_te1", "b_te1", "w_te2", "b_te2"):
        ref = sm.global_params(TINY_T)[name]
        np.testing.assert_array_equal(ctx.get_weight(mid, -1, name, ref.shape, ref.dtype), ref, err_msg=name)
    ctx.close()


def _oracle_params(shape):
    return sm.as_f64(sm.global_params(shape)), [sm.as_f64(sm.block_params(shape, l)) for l in range(shape.layers)]


@pytest.mark.parametrize("shape,grids", [
    (TINY_T.with_layers(1), [sm.token_grid(256, 256), sm.token_grid(384, 128)]),
    (sm.WAN_1_3B.with_layers(1).with_text(512, 4096), [sm.token_grid(512, 512), sm.token_grid(640, 384)]),
], ids=["tiny", "wan1.3b"])
def test_block_with_cross_attention_matches_oracle(gs, shape, grids):
    ctx = gs.Context(device=0)
    mid = _mk(ctx, shape)
    ns = [int(np.prod(g)) for g in grids]
    g = np.random.default_rng(3)
    x = g.standard_normal((sum(ns), shape.dim)).astype(np.float32)
    prompts = np.stack([sm.prompt_embeds(shape, 70 + r, 0) for r in range(len(ns))])
    ts = [900.0, 333.0]
    out = ctx.debug_block(mid, 0, x, grids, [0, 0], ns, ts, prompts=prompts)
    ctx.close()
    glob, blocks = _oracle_params(shape)
    e_req = np.stack([dit.time_embedding(np.float64(np.float32(t)), glob)[1] for t in ts])
    ctxs = [dit.text_embedding(rng.bf16_bits_to_f64(p), glob) for p in prompts]
    offs = np.cumsum([0] + ns[:-1])
    ref = dit.dit_block(x.astype(np.float64), blocks[0], e_req,
                        [(int(o), n, gr) for o, n, gr in zip(offs, ns, grids)], shape.heads, ctxs)
    for a, n in zip(offs, ns):
        err = rel_l2(out[a:a + n].astype(np.float64) - x[a:a + n], ref[a:a + n] - x[a:a + n])
        assert err < TOL, err


@pytest.mark.parametrize("cfg", [0.0, 1.5, 5.0])
def test_step_with_text_and_cfg_matches_oracle(gs, cfg):
    """One step.  With guidance the latent delta is dsig (g v_c - (g-1) v_u): bf16-level errors of
    the two branch velocities are amplified by the CFG condition number
    kappa = (g |v_c| + |g-1| |v_u|) / |v|, so the bar is TOL * kappa."""
    shape = TINY_T
    ctx = gs.Context(device=0)
    mid = _mk(ctx, shape)
    req = ctx.submit_text(mid, 256, 256, 1, 50, 1000, [0], prompt_seed=77, cfg_scale=cfg)
    z0 = ctx.read_latent(req)
    assert ctx.run_steps([req], [0], 1) == 1
    z1 = ctx.read_latent(req)
    ctx.close()
    glob, blocks = _oracle_params(shape)
    pc = rng.bf16_bits_to_f64(sm.prompt_embeds(shape, 77, 0))
    pu = rng.bf16_bits_to_f64(sm.prompt_embeds(shape, 77, 1)) if cfg > 0 else None
    ref = dit.dit_steps([z0.astype(np.float64)], [(1, 16, 16)], [0], 50, 1, glob, blocks, shape.heads,
                        prompts=[(pc, pu)], cfg=[cfg])[0]
    kappa = 1.0
    if cfg > 0:
        t0 = 1000.0 * dit.sigmas(50)[0]
        vc = dit.dit_velocity([z0.astype(np.float64)], [(1, 16, 16)], [t0], glob, blocks, shape.heads,
                              [dit.text_embedding(pc, glob)])[0]
        vu = dit.dit_velocity([z0.astype(np.float64)], [(1, 16, 16)], [t0], glob, blocks, shape.heads,
                              [dit.text_embedding(pu, glob)])[0]
        v = dit.cfg_velocity(vc, vu, cfg)
        kappa = (cfg * np.linalg.norm(vc) + abs(cfg - 1) * np.linalg.norm(vu)) / np.linalg.norm(v)
    err = rel_l2(z1.astype(np.float64) - z0, ref - z0)
    assert err < TOL * kappa, (err, kappa)


def test_seeded_prompt_equals_host_prompt_bitwise(gs):
    """The device prompt generator equals synth.rng's numpy generator bit for bit."""
    shape = TINY_T
    ctx = gs.Context(device=0)
    mid = _mk(ctx, shape)
    a = ctx.submit_text(mid, 256, 256, 1, 50, 1000, [0], prompt_seed=12, cfg_scale=4.0)
    host = np.stack([sm.prompt_embeds(shape, 12, 0), sm.prompt_embeds(shape, 12, 1)])
    b = ctx.submit_text(mid, 256, 256, 1, 50, 1000, [0], prompt_seed=999, cfg_scale=4.0, prompt_embeds=host)
    ctx.run_steps([a], [0], 1)
    ctx.run_steps([b], [0], 1)
    za, zb = ctx.read_latent(a), ctx.read_latent(b)
    ctx.close()
    assert np.array_equal(za.view(np.uint32), zb.view(np.uint32))


def _run(gs, shape, ranks_seq, k_seq, cfg=5.0, batch_with=None, world=8):
    ctx = gs.Context(device=0, world_size=world, emulated=True)
    mid = _mk(ctx, shape)
    req = ctx.submit_text(mid, 416, 240, 5, 50, 1000, ranks_seq[0], prompt_seed=5, cfg_scale=cfg)
    others = []
    if batch_with:
        others = [ctx.submit_text(mid, w, h, f, 50, 1001 + i, ranks_seq[0], prompt_seed=9 + i, cfg_scale=c)
                  for i, (w, h, f, c) in enumerate(batch_with)]
    for i, (ranks, k) in enumerate(zip(ranks_seq, k_seq)):
        if i:
            ctx.preempt(req)
            ctx.resume(req, ranks)
        assert ctx.run_steps([req] + (others if i == 0 else []), ranks, k) == k
    z = ctx.read_latent(req)
    ctx.close()
    return z


def test_text_cfg_bit_exact_across_sp_batching_and_resume(gs):
    shape = sm.WAN_1_3B.with_layers(1).with_text(512, 4096)
    ref = _run(gs, shape, [[0]], [2])
    for p in (2, 4, 8):
        z = _run(gs, shape, [list(range(p))], [2])
        assert np.array_equal(z.view(np.uint32), ref.view(np.uint32)), f"p={p}"
    z = _run(gs, shape, [[0]], [2], batch_with=[(256, 256, 1, 5.0), (416, 240, 5, 0.0)])
    assert np.array_equal(z.view(np.uint32), ref.view(np.uint32)), "batched"
    z = _run(gs, shape, [[0, 1, 2, 3], [6, 7]], [1, 1])
    assert np.array_equal(z.view(np.uint32), ref.view(np.uint32)), "preempt/resume"
    z = _run(gs, shape, [[0], [0]], [1, 1])
    assert np.array_equal(z.view(np.uint32), ref.view(np.uint32)), "k=2 in one call == 1 + 1"


def test_multi_step_cfg_matches_oracle(gs):
    """Three steps in one call: the CFG update must keep both branches on the same latent."""
    shape = TINY_T
    ctx = gs.Context(device=0)
    mid = _mk(ctx, shape)
    req = ctx.submit_text(mid, 256, 256, 1, 50, 1000, [0], prompt_seed=78, cfg_scale=2.0)
    z0 = ctx.read_latent(req)
    assert ctx.run_steps([req], [0], 3) == 3
    z3 = ctx.read_latent(req)
    ctx.close()
    glob, blocks = _oracle_params(shape)
    pc = rng.bf16_bits_to_f64(sm.prompt_embeds(shape, 78, 0))
    pu = rng.bf16_bits_to_f64(sm.prompt_embeds(shape, 78, 1))
    g = 2.0
    ctxc, ctxu = dit.text_embedding(pc, glob), dit.text_embedding(pu, glob)
    sig = dit.sigmas(50)
    z, bound = z0.astype(np.float64), 0.0
    for i in range(3):
        # DESIGN.md reading 21: the latent delta is sum_i dsig_i (g v_c,i - (g-1) v_u,i), so
        # per-branch velocity errors <= TOL |v| add up to TOL * sum_i |dsig_i| (g |v_c,i| +
        # |g-1| |v_u,i|): the bar is TOL * kappa with kappa that sum over |z3 - z0|.
        vc = dit.dit_velocity([z], [(1, 16, 16)], [1000.0 * sig[i]], glob, blocks, shape.heads, [ctxc])[0]
        vu = dit.dit_velocity([z], [(1, 16, 16)], [1000.0 * sig[i]], glob, blocks, shape.heads, [ctxu])[0]
        bound += abs(sig[i + 1] - sig[i]) * (g * np.linalg.norm(vc) + abs(g - 1) * np.linalg.norm(vu))
        z = dit.euler(z, dit.cfg_velocity(vc, vu, g), sig[i], sig[i + 1])
    ref = dit.dit_steps([z0.astype(np.float64)], [(1, 16, 16)], [0], 50, 3, glob, blocks, shape.heads,
                        prompts=[(pc, pu)], cfg=[g])[0]
    np.testing.assert_allclose(z, ref, rtol=0, atol=1e-12)   # the unrolled loop is dit_steps
    kappa = bound / np.linalg.norm(ref - z0)
    err = rel_l2(z3.astype(np.float64) - z0, ref - z0)
    assert err < TOL * kappa, (err, kappa)


def test_submit_contract_for_text_models(gs):
    ctx = gs.Context(device=0)
    mt = _mk(ctx, TINY_T)
    m0 = ctx.model_create(384, 6, 1536, 1)
    with pytest.raises(gs.GsError):
        ctx.submit(mt, 256, 256, 1, 50, 1, [0])          # text model needs a prompt
    with pytest.raises(gs.GsError):
        ctx.submit_text(m0, 256, 256, 1, 50, 1, [0])     # plain model has no cross-attention
    ctx.close()
