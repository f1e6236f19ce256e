"""Block / step parity against the fp64 oracle (rung T3) and GPU-vs-GPU bit-exactness (rung T4):
SP degree 1/2/4/8, batch composition, preempt -> re-shard -> resume.  Multi-rank cases use the
emulated context (W virtual ranks on the one GPU, exchanges as device copies; same kernels and
shard shapes as the NCCL path)."""
import threading

import numpy as np
import pytest

from oracle import dit
from synth import models as sm
from synth import rng
from tests.gpu_util import max_row_rel_l2, oracle_steps_per_request, rel_l2

pytestmark = pytest.mark.gpu

TOL = 1e-2  # BASELINE.json north_star: relative L2 vs the CPU oracle (bf16 storage, fp32 acc)


@pytest.fixture(scope="module")
def gs():
    import paper_2604_04335_b200 as m
    m.load()
    return m


def _mk(ctx, shape):
    return ctx.model_create(shape.dim, shape.heads, shape.ffn, shape.layers, shape.weight_seed)


def _block_case(ctx, shape, grids, ts, seed=11):
    """x_in random fp32 per request; returns (x_in, gpu_out, oracle_out)."""
    mid = _mk(ctx, shape)
    g = np.random.default_rng(seed)
    ns = [int(np.prod(gr)) for gr in grids]
    x = g.standard_normal((sum(ns), shape.dim)).astype(np.float32)
    out = ctx.debug_block(mid, 0, x, grids, [0] * len(ns), ns, ts)
    glob = sm.as_f64(sm.global_params(shape))
    blk = sm.as_f64(sm.block_params(shape, 0))
    e_req = np.stack([dit.time_embedding(np.float64(np.float32(t)), glob)[1] for t in ts])
    offs = np.cumsum([0] + ns[:-1])
    ref = dit.dit_block(x.astype(np.float64), blk, e_req,
                        [(int(o), n, gr) for o, n, gr in zip(offs, ns, grids)], shape.heads)
    return x, out, ref


def test_block_config1_tiny(gs):
    ctx = gs.Context(device=0)
    x, out, ref = _block_case(ctx, sm.TINY, [sm.token_grid(256, 256)], [860.5])
    err = rel_l2(out.astype(np.float64) - x, ref - x)
    ctx.close()
    assert err < TOL, err


@pytest.mark.parametrize("shape", [
    sm.ModelShape("d1024-h64", 1024, 16, 4096, 1),    # row kernels: a warp per row (VPL 8 / 4)
    sm.ModelShape("d2048-h128", 2048, 16, 2048, 1),   # two warps per row, largest VPL of that regime
    sm.ModelShape("d3072-h128", 3072, 24, 1024, 1),   # 256 threads per row (Wan2.2-5B width [ext])
    pytest.param(sm.ModelShape("d8192-h128", 8192, 64, 256, 1), marks=pytest.mark.slow),  # largest D
])
def test_block_row_kernel_regimes(gs, shape):
    """Block parity at model widths outside configs 1-4, covering every row-kernel shape (threads
    per row 32 / 64 / 256 and their largest register tiles); two ragged requests so some 8-row CTAs
    straddle a request boundary (per-row modulation loads) and others stage it per CTA."""
    ctx = gs.Context(device=0)
    grids = [sm.token_grid(96, 80), sm.token_grid(48, 48)]   # 30 + 9 rows
    x, out, ref = _block_case(ctx, shape, grids, [700.0, 120.0])
    ctx.close()
    offs = np.cumsum([0] + [int(np.prod(g)) for g in grids])
    for a, b in zip(offs[:-1], offs[1:]):
        err = rel_l2(out[a:b].astype(np.float64) - x[a:b], ref[a:b] - x[a:b])
        assert err < TOL, (shape.name, err)


def test_block_config2_wan13b_varlen(gs):
    # config 2b: varlen 4-image batch {1024^2, 1280x768, 768x1280, 1152x896}, Wan-1.3B block
    grids = [sm.token_grid(1024, 1024), sm.token_grid(1280, 768), sm.token_grid(768, 1280),
             sm.token_grid(1152, 896)]
    ctx = gs.Context(device=0)
    x, out, ref = _block_case(ctx, sm.WAN_1_3B.with_layers(1), grids, [999.0, 800.0, 500.0, 37.5])
    ctx.close()
    offs = np.cumsum([0] + [int(np.prod(g)) for g in grids])
    for a, b in zip(offs[:-1], offs[1:]):
        err = rel_l2(out[a:b].astype(np.float64) - x[a:b], ref[a:b] - x[a:b])
        assert err < TOL, err


def test_step_config1_tiny_12_layers(gs):
    shape = sm.TINY.with_layers(12)
    ctx = gs.Context(device=0)
    mid = _mk(ctx, shape)
    req = ctx.submit(mid, 256, 256, 1, 50, 1000, [0])
    z0 = ctx.read_latent(req)
    ctx.run_steps([req], [0], 1)
    ctx.run_steps([req], [0], 1)
    z2 = ctx.read_latent(req)
    ctx.close()
    glob = sm.as_f64(sm.global_params(shape))
    blocks = [sm.as_f64(sm.block_params(shape, l)) for l in range(12)]
    ref = dit.dit_steps([z0.astype(np.float64)], [(1, 16, 16)], [0], 50, 2, glob, blocks,
                        shape.heads)[0]
    err = rel_l2(z2.astype(np.float64) - z0, ref - z0)
    assert err < TOL, err


def test_step_batched_varlen_images_match_oracle(gs):
    shape = sm.TINY.with_layers(2)
    ctx = gs.Context(device=0)
    mid = _mk(ctx, shape)
    sizes = [(256, 256), (512, 256), (256, 384)]
    reqs = [ctx.submit(mid, w, h, 1, 30, 1000 + i, [0]) for i, (w, h) in enumerate(sizes)]
    # put the requests at different timesteps first
    ctx.run_steps([reqs[1]], [0], 3)
    z0 = [ctx.read_latent(r) for r in reqs]
    ctx.run_steps(reqs, [0], 1)
    z1 = [ctx.read_latent(r) for r in reqs]
    ctx.close()
    glob = sm.as_f64(sm.global_params(shape))
    blocks = [sm.as_f64(sm.block_params(shape, l)) for l in range(2)]
    grids = [sm.token_grid(w, h) for w, h in sizes]
    ref = dit.dit_steps([z.astype(np.float64) for z in z0], grids, [0, 3, 0], 30, 1, glob, blocks,
                        shape.heads)
    for a, b, r in zip(z0, z1, ref):
        assert rel_l2(b.astype(np.float64) - a, r - a) < TOL


@pytest.mark.slow
def test_step_config2_wan13b_full_depth(gs):
    """"Full-step parity at full depth is done at configs 1-2".  Config 2a: four
    1024^2 images (4 x 4096 tokens) batched at different timesteps through all 30 Wan-1.3B-shaped
    layers, one step, latent delta vs oracle dit_steps (48.7 TFLOP fp64 on the host)."""
    shape = sm.WAN_1_3B
    ctx = gs.Context(device=0)
    mid = _mk(ctx, shape)
    reqs = [ctx.submit(mid, 1024, 1024, 1, 50, 1000 + i, [0]) for i in range(4)]
    ctx.run_steps([reqs[1]], [0], 2)            # requests at step indices 0, 2, 0, 0 ...
    ctx.run_steps([reqs[3]], [0], 7)            # ... and 7
    z0 = [ctx.read_latent(r) for r in reqs]
    assert ctx.run_steps(reqs, [0], 1) == 1
    z1 = [ctx.read_latent(r) for r in reqs]
    ctx.close()
    grids = [sm.token_grid(1024, 1024)] * 4
    ref = oracle_steps_per_request(shape, z0, grids, [0, 2, 0, 7], 50, 1)
    for i, (a, b, r) in enumerate(zip(z0, z1, ref)):
        err = rel_l2(b.astype(np.float64) - a, r - a)
        worst = max_row_rel_l2(b.astype(np.float64) - a, r - a)
        print(f"config2 step request {i}: rel-L2 {err:.3e}, worst row {worst:.3e}")
        assert err < TOL, (i, err)


# ----------------------------------------------------------------------------- T4 bit-exactness
def _run_sp(gs, shape, width, height, frames, p, k, steps=50, seed=1000):
    ctx = gs.Context(device=0, world_size=8, emulated=True)
    mid = _mk(ctx, shape)
    ranks = list(range(p))
    req = ctx.submit(mid, width, height, frames, steps, seed, ranks)
    assert ctx.run_steps([req], ranks, k) == k
    z = ctx.read_latent(req)
    ctx.close()
    return z


@pytest.mark.parametrize("shape,w,h,f", [(sm.TINY.with_layers(2), 256, 256, 1),
                                         (sm.WAN_1_3B.with_layers(1), 416, 240, 5)])
def test_bit_exact_across_sp_degree(gs, shape, w, h, f):
    ref = _run_sp(gs, shape, w, h, f, 1, 2)
    for p in (2, 4, 8):
        z = _run_sp(gs, shape, w, h, f, p, 2)
        assert np.array_equal(z.view(np.uint32), ref.view(np.uint32)), f"p={p}"


def test_bit_exact_across_batch_composition(gs):
    shape = sm.TINY.with_layers(2)
    ctx = gs.Context(device=0)
    mid = _mk(ctx, shape)
    alone = ctx.submit(mid, 256, 256, 1, 50, 1000, [0])
    ctx.run_steps([alone], [0], 2)
    za = ctx.read_latent(alone)
    a = ctx.submit(mid, 512, 256, 1, 50, 1001, [0])
    b = ctx.submit(mid, 256, 256, 1, 50, 1000, [0])
    c = ctx.submit(mid, 384, 384, 1, 50, 1002, [0])
    ctx.run_steps([a, b, c], [0], 2)
    zb = ctx.read_latent(b)
    ctx.close()
    assert np.array_equal(za.view(np.uint32), zb.view(np.uint32))


def test_preempt_reshard_resume_bit_exact(gs):
    shape = sm.WAN_1_3B.with_layers(1)
    w, h, f = 416, 240, 5
    ctx = gs.Context(device=0, world_size=8, emulated=True)
    mid = _mk(ctx, shape)
    straight = ctx.submit(mid, w, h, f, 50, 1000, [0, 1, 2, 3])
    ctx.run_steps([straight], [0, 1, 2, 3], 3)
    z_ref = ctx.read_latent(straight)

    req = ctx.submit(mid, w, h, f, 50, 1000, [0, 1, 2, 3])
    assert ctx.run_steps([req], [0, 1, 2, 3], 1) == 1
    assert ctx.preempt(req) == 1
    assert ctx.query(req)["state"] == gs.REQ_PAUSED
    with pytest.raises(gs.GsError):
        ctx.run_steps([req], [0, 1, 2, 3], 1)          # paused: contract violation
    before = ctx.read_latent(req)
    ctx.resume(req, [6, 7])                             # SP 4 -> 2 on a different GPU set
    np.testing.assert_array_equal(ctx.read_latent(req), before)   # re-shard is a pure copy
    assert ctx.run_steps([req], [6, 7], 1) == 1
    ctx.resume(req, [0, 2, 4, 5, 1, 3, 6, 7])           # SP 2 -> 8, permuted set
    assert ctx.run_steps([req], [0, 2, 4, 5, 1, 3, 6, 7], 1) == 1
    z = ctx.read_latent(req)
    q = ctx.query(req)
    ctx.close()
    assert q["steps_done"] == 3
    assert np.array_equal(z.view(np.uint32), z_ref.view(np.uint32))


def test_preempt_from_another_thread_stops_at_step_boundary(gs):
    shape = sm.TINY.with_layers(12)
    ctx = gs.Context(device=0)
    mid = _mk(ctx, shape)
    req = ctx.submit(mid, 512, 512, 1, 1000, 1000, [0])
    done = {}

    def run():
        done["n"] = ctx.run_steps([req], [0], 900)

    th = threading.Thread(target=run)
    th.start()
    import time
    time.sleep(0.3)
    ctx.preempt(req)
    th.join()
    q = ctx.query(req)
    assert q["state"] == gs.REQ_PAUSED
    assert q["steps_done"] == done["n"] < 900
    # progress is never lost and the run continues exactly from the boundary
    ctx.resume(req, [0])
    ctx.run_steps([req], [0], 900 - done["n"])
    z = ctx.read_latent(req)
    ref = ctx.submit(mid, 512, 512, 1, 1000, 1000, [0])
    ctx.run_steps([ref], [0], 900)
    zr = ctx.read_latent(ref)
    ctx.close()
    assert np.array_equal(z.view(np.uint32), zr.view(np.uint32))


@pytest.mark.parametrize("p,ring", [(8, 2), (8, 4), (8, 8), (4, 2), (2, 2)])
def test_usp_hybrid_bit_exact_vs_sp1(gs, p, ring):
    """NEXT-2 USP hybrid (gs_set_option "usp_ring"): Ulysses over p / ring head groups x a ring of
    `ring` query chunks per head (K / V gathered in token order) gives the same bytes as SP = 1, and
    the exchanges run as transfer plans (every head is cut, so no peer-store path)."""
    shape = sm.WAN_1_3B.with_layers(2)
    w, h, f = 416, 240, 5
    z1 = _run_sp(gs, shape, w, h, f, 1, 2)
    ctx = gs.Context(device=0, world_size=8, emulated=True)
    ctx.set_option("usp_ring", ring)
    mid = _mk(ctx, shape)
    ranks = list(range(p))
    req = ctx.submit(mid, w, h, f, 50, 1000, ranks)
    st0 = ctx.stats()
    assert ctx.run_steps([req], ranks, 2) == 2
    st = ctx.stats()
    z = ctx.read_latent(req)
    ctx.close()
    assert st["a2a_plan"] > st0["a2a_plan"] and st["a2a_peer"] == st0["a2a_peer"]
    assert np.array_equal(z.view(np.uint32), z1.view(np.uint32))


def test_async_runs_on_disjoint_sets_concurrent_and_bit_exact(gs):
    """gs_run_steps_async: two SP groups ({0,1} and {2,3,4,5}) in flight together from one thread
    give the same bytes as serial runs; a run on a set overlapping an in-flight run is refused
    (GS_ESTATE: Eq. capacity, Alg.1 "no GPU overlap" P:498)."""
    shape = sm.WAN_1_3B.with_layers(2)
    w, h, f = 416, 240, 5
    ctx = gs.Context(device=0, world_size=8, emulated=True)
    mid = _mk(ctx, shape)
    a = ctx.submit(mid, w, h, f, 50, 1000, [0, 1])
    b = ctx.submit(mid, w, h, f, 50, 1001, [2, 3, 4, 5])
    c = ctx.submit(mid, 256, 256, 1, 50, 1002, [1])
    ta = ctx.run_steps_async([a], [0, 1], 3)
    tb = ctx.run_steps_async([b], [2, 3, 4, 5], 3)
    with pytest.raises(gs.GsError) as ei:
        ctx.run_steps_async([c], [1], 1)             # rank 1 belongs to ticket ta
    assert ei.value.code == gs.GS_ESTATE
    with pytest.raises(gs.GsError):
        ctx.resume(c, [5])                            # new rank 5 belongs to ticket tb
    assert ctx.wait(tb) == 3 and ctx.wait(ta) == 3
    with pytest.raises(gs.GsError):
        ctx.wait(ta)                                  # a ticket is waited for once
    za, zb = ctx.read_latent(a), ctx.read_latent(b)
    refs = []
    for seed in (1000, 1001):
        r = ctx.submit(mid, w, h, f, 50, seed, [0])
        assert ctx.run_steps([r], [0], 3) == 3
        refs.append(ctx.read_latent(r))
    ctx.close()
    assert np.array_equal(za.view(np.uint32), refs[0].view(np.uint32))
    assert np.array_equal(zb.view(np.uint32), refs[1].view(np.uint32))


def test_queued_submit_then_place(gs):
    """A request submitted without placement holds no GPU (state QUEUED, |X_r| = 0) until
    gs_place; placed on GPU 3 it steps exactly like a request submitted straight onto GPU 0."""
    shape = sm.TINY.with_layers(2)
    ctx = gs.Context(device=0, world_size=4, emulated=True)
    mid = _mk(ctx, shape)
    g = np.random.default_rng(4)
    z0 = g.standard_normal((256, 64)).astype(np.float32)
    q = ctx.submit(mid, 256, 256, 1, 50, 1000, None, init_latent=z0)
    assert ctx.query(q)["state"] == gs.REQ_QUEUED and ctx.query(q)["ranks"] == []
    with pytest.raises(gs.GsError):
        ctx.read_latent(q)
    with pytest.raises(gs.GsError):
        ctx.run_steps([q], [3], 1)
    ctx.place(q, [3])
    with pytest.raises(gs.GsError):
        ctx.place(q, [2])                             # already placed
    np.testing.assert_array_equal(ctx.read_latent(q), z0)
    assert ctx.run_steps([q], [3], 2) == 2
    d = ctx.submit(mid, 256, 256, 1, 50, 1000, [0], init_latent=z0)
    assert ctx.run_steps([d], [0], 2) == 2
    zq, zd = ctx.read_latent(q), ctx.read_latent(d)
    # noise-seeded queued request == noise-seeded direct request
    s1 = ctx.submit(mid, 256, 256, 1, 50, 77, None)
    ctx.place(s1, [2])
    s2 = ctx.submit(mid, 256, 256, 1, 50, 77, [1])
    n1, n2 = ctx.read_latent(s1), ctx.read_latent(s2)
    ctx.close()
    assert np.array_equal(zq.view(np.uint32), zd.view(np.uint32))
    assert np.array_equal(n1.view(np.uint32), n2.view(np.uint32))
    with pytest.raises(ValueError):
        gs.Context.__new__(gs.Context)._latent_arg(np.zeros(10), 256, 256, 1)


def test_preempt_async_run_from_same_thread(gs):
    """Preempting a request whose run is in flight (started with gs_run_steps_async) takes effect
    at the next step boundary; the steps run are reported by gs_wait and progress is kept."""
    shape = sm.TINY.with_layers(12)
    ctx = gs.Context(device=0)
    mid = _mk(ctx, shape)
    req = ctx.submit(mid, 512, 512, 1, 1000, 1000, [0])
    t = ctx.run_steps_async([req], [0], 900)
    import time
    time.sleep(0.3)
    assert not ctx.ticket_done(t)
    ctx.preempt(req)
    n = ctx.wait(t)
    q = ctx.query(req)
    ctx.close()
    assert 0 < n < 900 and q["steps_done"] == n and q["state"] == gs.REQ_PAUSED


def test_contract_errors(gs):
    ctx = gs.Context(device=0, world_size=4, emulated=True)
    mid = _mk(ctx, sm.TINY)
    with pytest.raises(gs.GsError) as e:
        ctx.submit(mid, 250, 256, 1, 50, 1, [0])
    assert e.value.code == gs.GS_EINVAL
    with pytest.raises(gs.GsError):
        ctx.submit(mid, 256, 256, 1, 50, 1, [0, 1, 2])       # p = 3
    with pytest.raises(gs.GsError):
        ctx.submit(mid, 256, 256, 1, 50, 1, [1, 1])          # duplicate GPU
    r = ctx.submit(mid, 256, 256, 1, 2, 1, [0, 1])
    with pytest.raises(gs.GsError) as e:
        ctx.run_steps([r], [0], 1)                            # wrong placement
    assert e.value.code == gs.GS_ESTATE
    with pytest.raises(gs.GsError):
        ctx.run_steps([r], [0, 1], 3)                         # k > remaining
    assert ctx.run_steps([r], [0, 1], 2) == 2
    assert ctx.query(r)["state"] == gs.REQ_DONE
    ctx.close()


# ----------------------------------------------------------------------------- fused exchange
def _run_mode(gs, shape, sizes, p, k, a2a):
    """Batch of requests (w, h, frames) placed on ranks 0..p-1, k steps with the given a2a mode;
    returns (latents, stats)."""
    ctx = gs.Context(device=0, world_size=8, emulated=True)
    ctx.set_option("a2a", a2a)
    mid = _mk(ctx, shape)
    ranks = list(range(p))
    reqs = [ctx.submit(mid, w, h, f, 50, 1000 + i, ranks) for i, (w, h, f) in enumerate(sizes)]
    ctx.run_steps([reqs[0]], ranks, 1)                   # different timesteps inside the batch
    assert ctx.run_steps(reqs, ranks, k) == k
    zs = [ctx.read_latent(r) for r in reqs]
    st = ctx.stats()
    ctx.close()
    return zs, st


@pytest.mark.parametrize("shape,sizes,p", [
    (sm.WAN_1_3B.with_layers(2), [(416, 240, 5)], 2),
    (sm.WAN_1_3B.with_layers(1), [(416, 240, 5), (256, 256, 1), (320, 192, 1)], 4),
    (sm.WAN_14B.with_layers(1), [(320, 176, 5)], 8),
])
def test_fused_peer_exchange_bit_exact_vs_transfer_plans(gs, shape, sizes, p):
    """Peer-store all-to-alls (pack kernel and attention epilogue writing the consumers' buffers,
    flag barriers) give the same bytes as the transfer-plan exchange, and actually ran."""
    z_peer, st_peer = _run_mode(gs, shape, sizes, p, 2, 1)
    z_plan, st_plan = _run_mode(gs, shape, sizes, p, 2, 0)
    assert st_peer["a2a_peer"] > 0 and st_peer["a2a_plan"] == 0
    assert st_plan["a2a_plan"] > 0 and st_plan["a2a_peer"] == 0
    for a, b in zip(z_peer, z_plan):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_fused_exchange_uneven_heads_uses_transfer_plans(gs):
    """p = 8 does not divide Wan-1.3B's 12 heads: the batch falls back to the balanced-unit
    transfer plans (reading 9), still bit-exact with SP = 1."""
    shape = sm.WAN_1_3B.with_layers(1)
    z8, st = _run_mode(gs, shape, [(416, 240, 5)], 8, 1, 1)
    z1, _ = _run_mode(gs, shape, [(416, 240, 5)], 1, 1, 1)
    assert st["a2a_plan"] > 0 and st["a2a_peer"] == 0
    assert np.array_equal(z8[0].view(np.uint32), z1[0].view(np.uint32))



# ----------------------------------------------------------------------------- degenerate sizes
def test_degenerate_sizes_tiny_requests_and_empty_shards(gs):
    """Degenerate cases: a 16x16 image is ONE token (attention returns v: pin P2 n=1), a 32x16
    image is two; at SP 4 / 8 most ranks hold zero rows of them (empty shards: M = 0 kernels are
    skipped, the exchange moves nothing for them).  The batch still matches the fp64 oracle and
    is bit-exact across SP degree and against each request run alone."""
    shape = sm.TINY.with_layers(2)
    sizes = [(16, 16, 1), (32, 16, 1), (48, 48, 1), (256, 256, 1)]
    glob = sm.as_f64(sm.global_params(shape))
    blocks = [sm.as_f64(sm.block_params(shape, l)) for l in range(shape.layers)]
    zs = {}
    for p in (1, 2, 4, 8):
        ctx = gs.Context(device=0, world_size=8, emulated=True)
        mid = _mk(ctx, shape)
        ranks = list(range(p))
        reqs = [ctx.submit(mid, w, h, f, 50, 1000 + i, ranks) for i, (w, h, f) in enumerate(sizes)]
        z0 = [ctx.read_latent(r) for r in reqs]
        assert ctx.run_steps(reqs, ranks, 1) == 1
        zs[p] = [ctx.read_latent(r) for r in reqs]
        ctx.close()
        if p == 1:
            grids = [sm.token_grid(w, h) for w, h, _ in sizes]
            assert [int(np.prod(g)) for g in grids] == [1, 2, 9, 256]
            ref = dit.dit_steps([z.astype(np.float64) for z in z0], grids, [0] * len(sizes), 50, 1, glob, blocks,
                                shape.heads)
            for a, b, r in zip(z0, zs[1], ref):
                assert rel_l2(b.astype(np.float64) - a, r - a) < TOL
    for p in (2, 4, 8):
        for a, b in zip(zs[p], zs[1]):
            assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), f"p={p}"
    ctx = gs.Context(device=0)
    mid = _mk(ctx, shape)
    one = ctx.submit(mid, 16, 16, 1, 50, 1000, [0])
    ctx.run_steps([one], [0], 1)
    z_alone = ctx.read_latent(one)
    ctx.close()
    assert np.array_equal(z_alone.view(np.uint32), zs[1][0].view(np.uint32))


def test_programmatic_dependent_launch_bit_exact(gs):
    """Programmatic dependent launch only moves each kernel's setup ahead of the previous kernel's
    drain (griddepcontrol.wait precedes every global access): SP 1 / SP 4 steps with a ragged batch
    give identical bytes with it on and off, over repeated runs."""
    shape = sm.WAN_1_3B.with_layers(2)
    sizes = [(416, 240, 5), (256, 256, 1), (48, 32, 1)]
    out = {}
    for pdl in (1, 0, 1):
        for p in (1, 4):
            ctx = gs.Context(device=0, world_size=8, emulated=True)
            ctx.set_option("pdl", pdl)
            mid = _mk(ctx, shape)
            ranks = list(range(p))
            reqs = [ctx.submit(mid, w, h, f, 50, 1000 + i, ranks) for i, (w, h, f) in enumerate(sizes)]
            ctx.run_steps([reqs[0]], ranks, 1)
            ctx.run_steps(reqs, ranks, 2)
            zs = [ctx.read_latent(r) for r in reqs]
            ctx.set_option("pdl", 1)
            ctx.close()
            ref = out.setdefault(p, zs)
            for a, b in zip(zs, ref):
                assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), (pdl, p)
    for a, b in zip(out[4], out[1]):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
