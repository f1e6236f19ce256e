"""NEXT-3 live: the SLO-aware scheduler (paper_2604_04335_b200/scheduler.py) drives the C-ABI on an
emulated 8-GPU context -- profiled T_step / T_img tables measured from this build, arrivals of
videos and images, Alg. 1 plans applied with gs_place / gs_preempt / gs_resume and
gs_run_steps_async.  Whatever the scheduler decides (preempt, re-shard, SP switching, batching),
every request must end bitwise equal to running it alone, uninterrupted, at SP = 1."""
import numpy as np
import pytest

from paper_2604_04335_b200 import scheduler as S
from synth import models as sm

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gs():
    import paper_2604_04335_b200 as m
    m.load()
    return m


def test_live_scheduler_mixed_trace_bit_exact(gs):
    vs, ims = sm.WAN_1_3B.with_layers(2), sm.TINY.with_layers(2)
    ctx = gs.Context(device=0, world_size=8, emulated=True)
    mv = ctx.model_create(vs.dim, vs.heads, vs.ffn, vs.layers, vs.weight_seed)
    mi = ctx.model_create(ims.dim, ims.heads, ims.ffn, ims.layers, ims.weight_seed)
    vres, ires = (416, 240, 5), (256, 256)
    prof = S.measure_profile(ctx, mv, mi, [vres], [ires], 8, batch_sizes=(1, 2, 4), image_steps=6)
    assert all(v > 0 for v in prof.t_step.values()) and all(v > 0 for v in prof.t_img.values())
    ts = prof.step(*vres, 1)
    ti = prof.img(1, *ires)
    # two videos with loose deadlines, then a burst of images with tight ones
    arr = [S.Video(0, 0.0, 60 * ts + 5.0, *vres, 24), S.Video(1, 0.0, 80 * ts + 5.0, *vres, 16)]
    arr += [S.Image(10 + i, 4 * ts, 4 * ts + 6 * ti + 2.0, *ires, 6) for i in range(6)]
    sch = S.LiveScheduler(ctx, prof, 8, mv, mi, round_steps=2, idle_s=0.5)
    out = sch.run(arr)
    assert out["requests"] == 8
    assert all(r.done_at is not None for r in sch.videos + sch.images)
    got = {("v", v.rid): ctx.read_latent(v.req) for v in sch.videos}
    got.update({("i", i.rid): ctx.read_latent(i.req) for i in sch.images})
    # references: alone, uninterrupted, SP = 1 (same seeds as LiveScheduler._submit)
    for v in sch.videos:
        r = ctx.submit(mv, v.w, v.h, v.frames, v.steps, 5000 + v.rid, [0])
        ctx.run_steps([r], [0], v.steps)
        assert np.array_equal(got[("v", v.rid)].view(np.uint32), ctx.read_latent(r).view(np.uint32)), v.rid
        ctx.release(r)
    for i in sch.images:
        r = ctx.submit(mi, i.w, i.h, 1, i.steps, 6000 + i.rid, [0])
        ctx.run_steps([r], [0], i.steps)
        assert np.array_equal(got[("i", i.rid)].view(np.uint32), ctx.read_latent(r).view(np.uint32)), i.rid
        ctx.release(r)
    ctx.close()
    print("live scheduler:", {k: v for k, v in out.items() if k != "log"})
    print("actions:", [e[:3] for e in out["log"]][:40])
