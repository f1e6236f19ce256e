"""SLO-aware step-level scheduler driving the C-ABI live.

Host policy only: it decides, at every round boundary, which GPU set each request holds next
(§4.4: the allocation X_r(t) -> X_r(t + D_round) expresses start, continue,
preempt, resume and reconfigure) and turns the plan into gs_* calls.  No DiT arithmetic runs here;
every step runs in libgs.so's kernels (gs_run_steps_async).

Pieces, each citing the passage it follows:
  * slack_v = D_v - t_now - S_v^rem * T_step(v)                        Eq. slack, §4.2
  * victims: running videos by descending slack, slack > 0 only, until enough GPUs are free
                                                                        P:336-338 §4.2
  * resume triggers: budget-tight (time to deadline <= estimated completion) or idle (no image
    arrival for `idle_s`)                                               P:345-353 §4.2
  * EDF batching of same-resolution images under a per-GPU budget g, deadline-checked through the
    profiled T_img(b, w, h), with a wait budget from the earliest deadline in the batch
                                                                        P:390-398 §4.3, Eq. image-value
  * video candidates (hold / continue / scale down / scale up / resume on a free pool), laxity
    l_v(c, t) = D_v - (t + S_v^rem T_step(p_c)), f_v(c) = 1 / (1 + |l|), recoverable = [l >= 0]
                                                                        Eq. video-value
  * Alg. 1: knapsack DP over the video groups with lexicographic (recoverable count, score) and
    no GPU overlap, then the best image plan for the GPUs left free     P:471-535 §4.4
Readings (DESIGN.md §"NEXT-3"): the DP state is the exact set of GPUs used (a bitmask over N <= 8
GPUs) so "no GPU overlap with previous selections" is checked exactly (the paper indexes the DP by
the GPU count b only); a hold candidate has value 0 and recoverable 0 ("A hold candidate
carries zero value"); an SP group is an aligned block {p k, ..., p k + p - 1} when one is free,
else any p free GPUs (bit-exactness does not depend on the set).

The T_step / T_img tables are measured from this build (`measure_profile`), not the paper's.
"""
from __future__ import annotations

import itertools
import time
from dataclasses import dataclass, field

P_DEGREES = (1, 2, 4, 8)   # P, P:92 Listing genserve-api "elastic_sp=[1,2,4,8]"


# ------------------------------------------------------------------------------ requests
@dataclass
class Image:
    rid: int                 # scheduler id
    arrival: float
    deadline: float          # absolute
    w: int
    h: int
    steps: int
    req: int | None = None   # gs_req once submitted
    gpu: int | None = None   # placed GPU while its batch runs
    done_at: float | None = None

    @property
    def res(self):
        return (self.w, self.h)


@dataclass
class Video:
    rid: int
    arrival: float
    deadline: float
    w: int
    h: int
    frames: int
    steps: int
    steps_done: int = 0
    gpus: tuple = ()         # current allocation X_v(t) (empty = paused or not started)
    paused: bool = False
    req: int | None = None
    done_at: float | None = None

    @property
    def steps_rem(self):
        return self.steps - self.steps_done

    @property
    def p(self):
        return len(self.gpus)


# ------------------------------------------------------------------------------ profile
@dataclass
class Profile:
    """Profiled latencies (the paper's Profiler; Tab. notation T_img, T_step)."""
    t_step: dict = field(default_factory=dict)   # (w, h, frames, p) -> seconds per denoising step
    t_img: dict = field(default_factory=dict)    # (b, w, h) -> seconds for a whole batch of b images

    def step(self, w, h, frames, p):
        return self.t_step[(w, h, frames, p)]

    def img(self, b, w, h):
        return self.t_img[(b, w, h)]

    def degrees(self, w, h, frames):
        return [p for p in P_DEGREES if (w, h, frames, p) in self.t_step]


def slack(v: Video, t: float, prof: Profile, p: int | None = None) -> float:
    """Eq. slack: D_v - t_now - S_v^rem * T_step(v) at SP degree p (default: current)."""
    p = p or v.p
    return v.deadline - t - v.steps_rem * prof.step(v.w, v.h, v.frames, p)


def select_victims(running: list[Video], t: float, prof: Profile, gpus_needed: int) -> list[Video]:
    """Preemption victims: running videos ranked by descending slack, non-positive slack
    excluded, taken until `gpus_needed` GPUs are freed (or no candidate is left)."""
    ranked = sorted((v for v in running if v.gpus and slack(v, t, prof) > 0),
                    key=lambda v: slack(v, t, prof), reverse=True)
    out, freed = [], 0
    for v in ranked:
        if freed >= gpus_needed:
            break
        out.append(v)
        freed += v.p
    return out


def resume_trigger(v: Video, t: float, prof: Profile, last_image_arrival: float, idle_s: float) -> str | None:
    """Resume policy for a paused video: 'budget' when the time left to the deadline falls
    to the estimated completion at the fastest profiled degree, 'idle' when no image arrived for
    idle_s seconds; else None."""
    best = min(prof.step(v.w, v.h, v.frames, p) for p in prof.degrees(v.w, v.h, v.frames))
    if v.deadline - t <= v.steps_rem * best:
        return "budget"
    if t - last_image_arrival >= idle_s:
        return "idle"
    return None


# ------------------------------------------------------------------------------ images
def edf_batch(images: list[Image], g: int, t: float, prof: Profile, max_batch: int = 8):
    """EdfBatch(I(t), g) of Alg. 1 line 3 (Eq. image-value): up to g GPUs, each
    running one batch of same-resolution images formed in earliest-deadline-first order; an image
    joins a batch only if every member still meets its deadline with the enlarged batch
    (completion t + T_img(b)).  Returns (batches [(images)], recoverable count, score)."""
    pending = sorted(images, key=lambda i: (i.deadline, i.arrival, i.rid))
    batches, used = [], set()
    for _ in range(g):
        seed = next((i for i in pending if i.rid not in used and t + prof.img(1, i.w, i.h) <= i.deadline), None)
        if seed is None:
            seed = next((i for i in pending if i.rid not in used), None)  # late anyway: still serve EDF
        if seed is None:
            break
        batch = [seed]
        used.add(seed.rid)
        for c in pending:
            if c.rid in used or c.res != seed.res or len(batch) >= max_batch:
                continue
            if (1 + len(batch), c.w, c.h) not in prof.t_img:
                continue
            done = t + prof.img(len(batch) + 1, c.w, c.h)
            if all(done <= m.deadline for m in batch + [c]):
                batch.append(c)
                used.add(c.rid)
        batches.append(batch)
    rec, score = 0, 0.0
    for b in batches:
        done = t + prof.img(len(b), b[0].w, b[0].h)
        for i in b:
            s = i.deadline - done
            if s >= 0:
                rec += 1
                score += 1.0 / (1.0 + max(0.0, s))
    return batches, rec, score


def wait_budget(batch: list[Image], t: float, prof: Profile) -> float:
    """Dynamic wait budget: how long a batch may wait for more same-resolution requests
    and still meet the earliest deadline in it at the next batch size."""
    b = len(batch)
    key = (b + 1, batch[0].w, batch[0].h)
    lat = prof.t_img[key] if key in prof.t_img else prof.img(b, batch[0].w, batch[0].h)
    return max(0.0, min(i.deadline for i in batch) - t - lat)


# ------------------------------------------------------------------------------ videos
@dataclass
class Cand:
    video: Video
    kind: str                # hold | continue | down | up | resume | start
    gpus: tuple
    lax: float
    score: float
    recoverable: int

    @property
    def w(self):
        return len(self.gpus)

    @property
    def mask(self):
        m = 0
        for g in self.gpus:
            m |= 1 << g
        return m


def _groups(p: int, pool: set, n: int):
    """GPU sets of size p from `pool`: aligned blocks {p k .. p k + p - 1} first, then (if none)
    the lowest p free GPUs."""
    out = []
    for k in range(n // p):
        blk = tuple(range(p * k, p * k + p))
        if set(blk) <= pool:
            out.append(blk)
    if not out and len(pool) >= p:
        out.append(tuple(sorted(pool)[:p]))
    return out


def video_candidates(v: Video, t: float, prof: Profile, free: set, n: int) -> list[Cand]:
    """GenVideoCandidates (Alg. 1 line 5): hold; continue on X_v(t); scale down to a half
    of X_v(t); scale up onto X_v(t) plus free GPUs; resume / start on a free pool at every profiled
    degree.  Laxity l = D_v - (t + S_rem T_step(p)), f = 1 / (1 + |l|), recoverable = [l >= 0]."""
    degs = prof.degrees(v.w, v.h, v.frames)
    cands = [Cand(v, "hold", (), v.deadline - float("inf"), 0.0, 0)]

    def mk(kind, gpus):
        lax = v.deadline - (t + v.steps_rem * prof.step(v.w, v.h, v.frames, len(gpus)))
        return Cand(v, kind, tuple(gpus), lax, 1.0 / (1.0 + abs(lax)), int(lax >= 0))

    if v.gpus and not v.paused:
        cands.append(mk("continue", v.gpus))
        if v.p > 1 and v.p // 2 in degs:
            cands.append(mk("down", v.gpus[:v.p // 2]))
        if 2 * v.p in degs:
            for extra in _groups(v.p, free, n):
                cands.append(mk("up", tuple(v.gpus) + extra))
    else:
        pool = set(free) | set(v.gpus)
        for p in degs:
            for g in _groups(p, pool, n):
                cands.append(mk("resume" if v.steps_done else "start", g))
    return cands


@dataclass
class Plan:
    videos: dict                       # rid -> Cand
    image_batches: list                # [(gpu, [Image])]
    recoverable: int
    score: float


def dp_schedule(videos: list[Video], images: list[Image], t: float, prof: Profile, n: int,
                busy: set = frozenset()) -> Plan:
    """Alg. 1.  Stage 1: image candidates for every budget g and video candidates.
    Stage 2: DP over the video groups; the state is the exact mask of GPUs taken, the value the
    lexicographic (recoverable count, score) of Eq. dp-transition.  Stage 3: every terminal state is
    combined with the best image plan on its free GPUs; backtrack the best.  GPUs in `busy` (image
    batches still running) are outside G for this round."""
    avail = set(range(n)) - set(busy)
    img_c = {g: edf_batch(images, g, t, prof) for g in range(len(avail) + 1)}
    groups = [[c for c in video_candidates(v, t, prof, avail - set(v.gpus), n) if set(c.gpus) <= avail]
              for v in videos]
    NEG = (-1, -1.0)
    dp = [{0: ((0, 0.0), None)}]       # per stage: mask -> (value, (prev mask, cand))
    for cands in groups:
        nxt = {}
        for mask, (val, _bp) in dp[-1].items():
            for c in cands:
                if c.mask & mask:
                    continue                     # no GPU overlap with previous selections
                m2 = mask | c.mask
                v2 = (val[0] + c.recoverable, val[1] + c.score)
                if v2 > nxt.get(m2, (NEG, None))[0]:
                    nxt[m2] = (v2, (mask, c))
        dp.append(nxt)
    best = None
    for mask, (val, _bp) in dp[-1].items():
        free = sorted(avail - {g for g in range(n) if mask >> g & 1})
        batches, rec, score = img_c[len(free)]
        tot = (val[0] + rec, val[1] + score)
        if best is None or tot > best[0]:
            best = (tot, mask, free, batches)
    (rec, score), mask, free, batches = best
    chosen = {}
    for j in range(len(groups), 0, -1):
        _val, (pm, c) = dp[j][mask]
        chosen[c.video.rid] = c
        mask = pm
    return Plan(chosen, list(zip(free, batches)), rec, score)


def brute_force_schedule(videos, images, t, prof, n, busy=frozenset()):
    """Exhaustive reference of dp_schedule for small instances (tests): every combination of one
    candidate per video with pairwise disjoint GPU sets, plus the image plan on the rest."""
    avail = set(range(n)) - set(busy)
    groups = [[c for c in video_candidates(v, t, prof, avail - set(v.gpus), n) if set(c.gpus) <= avail]
              for v in videos]
    best = None
    for combo in itertools.product(*groups):
        used = set()
        ok = True
        for c in combo:
            if used & set(c.gpus):
                ok = False
                break
            used |= set(c.gpus)
        if not ok:
            continue
        free = avail - used
        _b, rec, score = edf_batch(images, len(free), t, prof)
        tot = (sum(c.recoverable for c in combo) + rec, sum(c.score for c in combo) + score)
        if best is None or tot > best:
            best = tot
    return best


# ------------------------------------------------------------------------------ live driver
def measure_profile(ctx, video_model, image_model, video_res, image_res, n, batch_sizes=(1, 2, 4),
                    image_steps=4, reps=2):
    """Profiled T_step / T_img tables measured from this build in the executing context (the
    paper's offline Profiler): median wall time of `reps` runs per configuration."""
    prof = Profile()
    for (w, h, f) in video_res:
        for p in P_DEGREES:
            if p > n:
                continue
            ranks = list(range(p))
            r = ctx.submit(video_model, w, h, f, 1000, 1, ranks)
            ctx.run_steps([r], ranks, 1)
            ts = []
            for _ in range(reps):
                a = time.perf_counter()
                ctx.run_steps([r], ranks, 1)
                ts.append(time.perf_counter() - a)
            ctx.release(r)
            prof.t_step[(w, h, f, p)] = sorted(ts)[len(ts) // 2]
    for (w, h) in image_res:
        for b in batch_sizes:
            ts = []
            for _ in range(reps):
                rs = [ctx.submit(image_model, w, h, 1, image_steps, 100 + i, [0]) for i in range(b)]
                a = time.perf_counter()
                ctx.run_steps(rs, [0], image_steps)
                ts.append(time.perf_counter() - a)
                for r in rs:
                    ctx.release(r)
            prof.t_img[(b, w, h)] = sorted(ts)[len(ts) // 2]
    return prof


class LiveScheduler:
    """Round-based serving loop over one gs context with n GPUs (ranks): at every round boundary it
    admits arrivals, computes Alg. 1's plan, applies it through gs_preempt / gs_resume / gs_place
    and starts the rounds' runs with gs_run_steps_async (videos: D_round steps; image batches: to
    completion), then waits for the videos' runs (the next boundary).  Records every scheduling
    action and each request's completion time."""

    def __init__(self, ctx, prof: Profile, n: int, video_model: int, image_model: int,
                 round_steps: int = 1, idle_s: float = 1.0, clock=time.perf_counter):
        self.ctx, self.prof, self.n = ctx, prof, n
        self.vm, self.im = video_model, image_model
        self.round_steps, self.idle_s, self.clock = round_steps, idle_s, clock
        self.videos: list[Video] = []
        self.images: list[Image] = []
        self.img_runs = []            # (ticket, gpu, [Image])
        self.log = []
        self.t0 = None
        self.last_img_arrival = 0.0

    def now(self):
        return self.clock() - self.t0

    def _submit(self, r):
        if isinstance(r, Video):
            r.req = self.ctx.submit(self.vm, r.w, r.h, r.frames, r.steps, 5000 + r.rid, None)
            self.videos.append(r)
        else:
            r.req = self.ctx.submit(self.im, r.w, r.h, 1, r.steps, 6000 + r.rid, None)
            self.images.append(r)
            self.last_img_arrival = r.arrival

    def _reap_images(self):
        keep = []
        for tk, gpu, batch in self.img_runs:
            if self.ctx.ticket_done(tk):
                self.ctx.wait(tk)
                for i in batch:
                    i.done_at = self.now()
                self.log.append((self.now(), "image_batch_done", gpu, [i.rid for i in batch]))
            else:
                keep.append((tk, gpu, batch))
        self.img_runs = keep

    def run(self, arrivals, max_rounds=10000):
        """arrivals: list of Image / Video with .arrival in seconds from the start."""
        pending = sorted(arrivals, key=lambda r: r.arrival)
        self.t0 = self.clock()
        for _ in range(max_rounds):
            t = self.now()
            while pending and pending[0].arrival <= t:
                self._submit(pending.pop(0))
            self._reap_images()
            live_v = [v for v in self.videos if v.done_at is None]
            queued_i = [i for i in self.images if i.gpu is None]
            if not pending and not live_v and not queued_i and not self.img_runs:
                break
            busy = {g for _tk, g, _b in self.img_runs}
            plan = dp_schedule(live_v, queued_i, t, self.prof, self.n, busy)
            tickets = self._apply(plan, t)
            if not tickets and not self.img_runs and pending:
                time.sleep(max(0.0, min(0.05, pending[0].arrival - self.now())))
            elif not tickets:
                time.sleep(0.005)
            for v, tk in tickets:
                n_run = self.ctx.wait(tk)
                v.steps_done += n_run
                if v.steps_rem == 0:
                    v.done_at = self.now()
                    self.log.append((v.done_at, "video_done", v.rid, v.gpus))
        self._reap_images()
        for tk, _g, batch in self.img_runs:
            self.ctx.wait(tk)
            for i in batch:
                i.done_at = self.now()
        return self.summary()

    def _apply(self, plan: Plan, t: float):
        ctx = self.ctx
        tickets = []
        # videos: hold -> pause; a new GPU set -> resume / reconfigure (re-shard); start -> place
        for v in [v for v in self.videos if v.done_at is None]:
            c = plan.videos.get(v.rid)
            if c is None:
                continue
            if c.kind == "hold":
                if v.gpus and not v.paused:
                    ctx.preempt(v.req)
                    self.log.append((t, "preempt", v.rid, v.gpus))
                v.paused = True
                continue
            if c.kind == "start":
                ctx.place(v.req, list(c.gpus))
                self.log.append((t, "start", v.rid, c.gpus))
            elif tuple(c.gpus) != tuple(v.gpus) or v.paused:
                if v.gpus and not v.paused:
                    ctx.preempt(v.req)
                ctx.resume(v.req, list(c.gpus))
                self.log.append((t, c.kind if c.kind != "continue" else "resume", v.rid, c.gpus))
            v.gpus, v.paused = tuple(c.gpus), False
        for gpu, batch in plan.image_batches:
            for i in batch:
                ctx.place(i.req, [gpu])
                i.gpu = gpu
            self.log.append((t, "image_batch", gpu, [i.rid for i in batch]))
            tk = ctx.run_steps_async([i.req for i in batch], [gpu], batch[0].steps)
            self.img_runs.append((tk, gpu, batch))
        for v in self.videos:
            if v.done_at is None and v.gpus and not v.paused:
                k = min(self.round_steps, v.steps_rem)
                tickets.append((v, ctx.run_steps_async([v.req], list(v.gpus), k)))
        return tickets

    def summary(self):
        reqs = self.videos + self.images
        met = [r for r in reqs if r.done_at is not None and r.done_at <= r.deadline]
        return {"requests": len(reqs), "met": len(met),
                "slo_attainment": len(met) / max(len(reqs), 1),
                "actions": sum(1 for e in self.log if e[1] in ("preempt", "resume", "down", "up")),
                "log": self.log}
