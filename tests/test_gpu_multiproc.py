"""Multi-process NCCL path (one process per GPU): needs >= 2 GPUs and skips below.

Two processes with one context each (NCCL world of 2) run a Wan-1.3B-shaped request at SP = 2 with
the fused peer-store exchange (CUDA IPC mappings, flag barriers) and with the NCCL transfer plans,
re-shard it SP 2 -> 1 -> 2 by NCCL point-to-point (gs_resume), resume a request onto the rank that
did not hold it, and preempt from one process only (the per-step agree_stop exchange makes both stop
at the same boundary).  Every result must equal the single-process emulated run bit for bit.
(tools/mp_nccl_check.py is the stand-alone version.)"""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ndev():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


needs2 = pytest.mark.skipif(_ndev() < 2, reason="multi-process NCCL path needs >= 2 GPUs (one process per GPU)")


def _worker(rank, uid, q):
    try:
        sys.path.insert(0, ROOT)
        import paper_2604_04335_b200 as gs
        from synth import models as sm
        shape = sm.WAN_1_3B.with_layers(2)
        out = {}
        ctx = gs.Context(device=rank, world_size=2, rank=rank, nccl_uid=uid)
        mid = ctx.model_create(shape.dim, shape.heads, shape.ffn, shape.layers, shape.weight_seed)
        for mode in (1, 0):                          # peer stores, transfer plans
            ctx.set_option("a2a", mode)
            st0 = ctx.stats()
            req = ctx.submit(mid, 416, 240, 5, 50, 1000, [0, 1])
            assert ctx.run_steps([req], [0, 1], 2) == 2
            z = ctx.read_latent(req)
            ctx.release(req)
            st = ctx.stats()
            out[f"mode{mode}"] = (z.tobytes(), st["a2a_peer"] - st0["a2a_peer"], st["a2a_plan"] - st0["a2a_plan"])
        # re-shard SP 2 -> 1 (onto rank 0) -> 2 with a step at each placement
        req = ctx.submit(mid, 416, 240, 5, 50, 1001, [0, 1])
        ctx.run_steps([req], [0, 1], 1)
        ctx.resume(req, [0])
        if rank == 0:
            ctx.run_steps([req], [0], 1)
        ctx.resume(req, [0, 1])
        ctx.run_steps([req], [0, 1], 1)
        out["reshard"] = ctx.read_latent(req).tobytes()
        ctx.release(req)
        # a request placed on rank 0 only, resumed onto rank 1 (rank 1's process never held a shard)
        req = ctx.submit(mid, 416, 240, 5, 50, 1002, [0])
        if rank == 0:
            ctx.run_steps([req], [0], 1)
        ctx.resume(req, [1])
        if rank == 1:
            ctx.run_steps([req], [1], 1)
        out["move"] = ctx.read_latent(req).tobytes()
        ctx.release(req)
        # preempt from rank 0 only, mid-run: both processes stop at the same step boundary
        req = ctx.submit(mid, 416, 240, 5, 1000, 1003, [0, 1])
        t = ctx.run_steps_async([req], [0, 1], 500)
        if rank == 0:
            import time
            time.sleep(0.5)
            ctx.preempt(req)
        out["stopped_at"] = ctx.wait(t)
        ctx.close()
        q.put((rank, out, None))
    except Exception as e:  # noqa: BLE001
        import traceback
        q.put((rank, None, f"{e!r}\n{traceback.format_exc()}"))


@needs2
def test_two_process_sp2_peer_plans_reshard_preempt_bit_exact():
    import torch.multiprocessing as mp

    import paper_2604_04335_b200 as gs
    from synth import models as sm
    uid = gs.nccl_unique_id()
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    ps = [ctxm.Process(target=_worker, args=(r, uid, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(2):
        r, v, err = q.get(timeout=900)
        assert err is None, f"rank {r}: {err}"
        res[r] = v
    for p in ps:
        p.join(timeout=60)
    shape = sm.WAN_1_3B.with_layers(2)
    ctx = gs.Context(device=0, world_size=2, emulated=True)
    mid = ctx.model_create(shape.dim, shape.heads, shape.ffn, shape.layers, shape.weight_seed)
    r0 = ctx.submit(mid, 416, 240, 5, 50, 1000, [0, 1])
    ctx.run_steps([r0], [0, 1], 2)
    zref = ctx.read_latent(r0)
    r1 = ctx.submit(mid, 416, 240, 5, 50, 1001, [0])
    ctx.run_steps([r1], [0], 3)
    zres = ctx.read_latent(r1)
    r2 = ctx.submit(mid, 416, 240, 5, 50, 1002, [0])
    ctx.run_steps([r2], [0], 2)
    zmove = ctx.read_latent(r2)
    ctx.close()
    n = zref.shape[0]

    def gather(key, halves=True):
        z = np.zeros_like(zref)
        for r in range(2):
            zr = np.frombuffer(res[r][key] if not isinstance(res[r][key], tuple) else res[r][key][0],
                               dtype=np.float32).reshape(zref.shape)
            lo, hi = (r * n // 2, (r + 1) * n // 2) if halves else (0, n)
            if halves or r == 1:
                z[lo:hi] = zr[lo:hi]
        return z

    for mode in (1, 0):
        assert np.array_equal(gather(f"mode{mode}").view(np.uint32), zref.view(np.uint32)), mode
    assert res[0]["mode1"][1] > 0, "peer-store exchange did not run"
    assert res[0]["mode0"][2] > 0, "transfer plans did not run"
    assert np.array_equal(gather("reshard").view(np.uint32), zres.view(np.uint32))
    assert np.array_equal(gather("move", halves=False).view(np.uint32), zmove.view(np.uint32))
    assert res[0]["stopped_at"] == res[1]["stopped_at"] < 500
