"""NEXT-3 scheduler policy (paper_2604_04335_b200/scheduler.py) on the host: Eq. slack, victim
choice, resume triggers, EDF batching, and Alg. 1's DP pinned against exhaustive search; the live
loop against a recording fake context (the GPU version is tests/test_gpu_scheduler.py)."""
import random

import pytest

from paper_2604_04335_b200 import scheduler as S


def _prof():
    p = S.Profile()
    for p_ in (1, 2, 4, 8):
        p.t_step[(1280, 720, 81, p_)] = 8.0 / p_ ** 0.9      # sub-linear SP speed-up
        p.t_step[(832, 480, 81, p_)] = 3.0 / p_ ** 0.8
    for b in range(1, 9):
        p.t_img[(b, 1024, 1024)] = 2.0 + 0.9 * (b - 1)
        p.t_img[(b, 512, 512)] = 0.6 + 0.25 * (b - 1)
    return p


def test_slack_is_eq_slack():
    """slack_v = D_v - t_now - S_rem * T_step(v), by hand."""
    prof = _prof()
    v = S.Video(1, 0.0, 500.0, 1280, 720, 81, 50, steps_done=20, gpus=(0, 1, 2, 3))
    assert S.slack(v, 100.0, prof) == pytest.approx(500.0 - 100.0 - 30 * 8.0 / 4 ** 0.9)
    assert S.slack(v, 100.0, prof, p=8) == pytest.approx(400.0 - 30 * 8.0 / 8 ** 0.9)


def test_victims_descending_slack_positive_only():
    """highest slack first, non-positive slack never preempted, stop once enough GPUs."""
    prof = _prof()
    t = 0.0
    a = S.Video(1, 0, 1000.0, 1280, 720, 81, 50, gpus=(0, 1))          # large slack
    b = S.Video(2, 0, 300.0, 1280, 720, 81, 50, gpus=(2, 3))           # smaller slack
    c = S.Video(3, 0, 10.0, 1280, 720, 81, 50, gpus=(4, 5, 6, 7))      # negative slack
    assert [v.rid for v in S.select_victims([a, b, c], t, prof, 2)] == [1]
    assert [v.rid for v in S.select_victims([a, b, c], t, prof, 3)] == [1, 2]
    assert [v.rid for v in S.select_victims([a, b, c], t, prof, 8)] == [1, 2]   # c excluded


def test_resume_triggers():
    """budget-tight when the time left <= completion at the fastest degree; idle after a
    quiet period; otherwise stay paused."""
    prof = _prof()
    v = S.Video(1, 0, 100.0, 1280, 720, 81, 50, steps_done=10, paused=True)
    fastest = 40 * 8.0 / 8 ** 0.9
    assert S.resume_trigger(v, 100.0 - fastest - 1.0, prof, 99.0, 5.0) is None
    assert S.resume_trigger(v, 100.0 - fastest + 1e-9, prof, 0.0, 1e9) == "budget"
    assert S.resume_trigger(v, 10.0, prof, 2.0, 5.0) == "idle"


def test_edf_batches_meet_deadlines_and_respect_resolution():
    prof = _prof()
    imgs = [S.Image(i, 0.0, d, 1024, 1024, 50) for i, d in enumerate([3.0, 4.0, 5.2, 30.0, 30.0])]
    imgs += [S.Image(10 + i, 0.0, 2.0, 512, 512, 50) for i in range(3)]
    batches, rec, _score = S.edf_batch(imgs, 2, 0.0, prof)
    for b in batches:
        assert len({i.res for i in b}) == 1
    # EDF: the 512^2 images (deadline 2.0) seed the first batch; all three fit (0.6 + 2 * 0.25 = 1.1)
    assert sorted(i.rid for i in batches[0]) == [10, 11, 12]
    # second GPU: 1024^2 from deadline 3.0; b = 2 completes at 2.9 <= 3.0 ok, b = 3 at 3.8 > 3.0
    assert sorted(i.rid for i in batches[1]) == [0, 1]
    assert rec == 5
    assert S.wait_budget(batches[1], 0.0, prof) == 0.0   # b = 3 would miss deadline 3.0
    assert S.wait_budget([imgs[3]], 0.0, prof) == pytest.approx(30.0 - 2.9)


def _random_instance(rng, n=8):
    prof = _prof()
    res = [(1280, 720, 81), (832, 480, 81)]
    vids, used = [], set()
    for k in range(rng.randint(1, 3)):
        w, h, f = rng.choice(res)
        state = rng.choice(["run", "paused", "new"])
        gpus = ()
        if state == "run":
            for p in (4, 2, 1):
                blocks = [tuple(range(p * i, p * i + p)) for i in range(n // p)]
                free = [b for b in blocks if not used & set(b)]
                if free:
                    gpus = rng.choice(free)
                    used |= set(gpus)
                    break
        v = S.Video(k, 0.0, rng.uniform(20, 400), w, h, f, 50, steps_done=rng.randint(0, 40),
                    gpus=gpus, paused=state == "paused")
        if state == "new":
            v.steps_done = 0
        vids.append(v)
    imgs = [S.Image(100 + i, 0.0, rng.uniform(1.5, 12), *rng.choice([(1024, 1024), (512, 512)]), 50)
            for i in range(rng.randint(0, 6))]
    return prof, vids, imgs


def test_dp_equals_exhaustive_search():
    """Alg. 1's DP reaches the same lexicographic optimum (recoverable count, score) as
    enumerating every disjoint combination of candidates (plus the image plan on the free GPUs)."""
    rng = random.Random(7)
    for _ in range(60):
        prof, vids, imgs = _random_instance(rng)
        t = rng.uniform(0, 10)
        busy = set(rng.sample(range(8), rng.randint(0, 2))) - {g for v in vids for g in v.gpus}
        plan = S.dp_schedule(vids, imgs, t, prof, 8, busy)
        best = S.brute_force_schedule(vids, imgs, t, prof, 8, busy)
        assert plan.recoverable == best[0]
        assert plan.score == pytest.approx(best[1], rel=1e-12, abs=1e-12)
        # the plan is feasible: disjoint GPU sets, capacity (Eq. capacity), busy avoided
        taken = [g for c in plan.videos.values() for g in c.gpus] + [g for g, _b in plan.image_batches]
        assert len(taken) == len(set(taken)) and len(taken) <= 8 and not set(taken) & busy


def test_dp_preempts_high_slack_video_for_urgent_images():
    """An 8-GPU video with ample slack yields GPUs to four urgent images (the Fig. preemption
    scenario): the DP scales it down (or holds it) and serves the images."""
    prof = _prof()
    v = S.Video(1, 0.0, 2000.0, 1280, 720, 81, 50, steps_done=5, gpus=tuple(range(8)))
    imgs = [S.Image(10 + i, 0.0, 3.0, 1024, 1024, 50) for i in range(4)]
    plan = S.dp_schedule([v], imgs, 0.0, prof, 8)
    assert plan.recoverable == 5
    assert plan.videos[1].kind in ("down", "hold") and len(plan.image_batches) >= 2


class FakeCtx:
    """Records gs_* calls; runs complete instantly (steps counted)."""

    def __init__(self):
        self.calls = []
        self.next = 1
        self.tickets = {}

    def submit(self, model, w, h, f, steps, seed, ranks, init_latent=None):
        self.calls.append(("submit", w, h, f, ranks))
        self.next += 1
        return self.next

    def place(self, req, ranks):
        self.calls.append(("place", req, tuple(ranks)))

    def preempt(self, req):
        self.calls.append(("preempt", req))

    def resume(self, req, ranks):
        self.calls.append(("resume", req, tuple(ranks)))

    def run_steps_async(self, reqs, ranks, k):
        self.next += 1
        self.tickets[self.next] = k
        self.calls.append(("run", tuple(reqs), tuple(ranks), k))
        return self.next

    def ticket_done(self, t):
        return True

    def wait(self, t):
        return self.tickets.pop(t)


def test_live_loop_actions_on_fake_context():
    """The live loop turns plans into gs_* calls: a video starts on an SP group, images arriving
    later are batched on free GPUs (placed, run to completion), and every request finishes."""
    prof = _prof()
    fake = FakeCtx()
    clock = {"t": 0.0}

    def tick():
        clock["t"] += 0.5
        return clock["t"]

    sch = S.LiveScheduler(fake, prof, 8, 0, 1, round_steps=5, clock=tick)
    arr = [S.Video(1, 0.0, 500.0, 1280, 720, 81, 20)]
    arr += [S.Image(10 + i, 1.0, 30.0, 1024, 1024, 50) for i in range(3)]
    out = sch.run(arr)
    assert out["requests"] == 4 and all(r.done_at is not None for r in sch.videos + sch.images)
    kinds = [c[0] for c in fake.calls]
    assert "place" in kinds and "run" in kinds
    vid_runs = [c for c in fake.calls if c[0] == "run" and c[1] == (sch.videos[0].req,)]
    assert sum(c[3] for c in vid_runs) == 20          # progress accounted step by step
