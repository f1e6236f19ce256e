"""Two real processes (one context each, NCCL world of 2) running a Wan-1.3B-shaped request at
SP = 2 with the fused peer-store exchange (CUDA IPC mappings, flag barriers) and with the NCCL
transfer plans; both must equal the single-process emulated SP = 2 run bit for bit.  On a box with
one GPU both processes share device 0 (when NCCL accepts that); otherwise devices 0 and 1.
  python tools/mp_nccl_check.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(rank, world, uid, dev, q):
    try:
        import numpy as np
        import paper_2604_04335_b200 as gs
        from synth import models as sm
        shape = sm.WAN_1_3B.with_layers(2)
        out = {}
        ctx = gs.Context(device=dev[rank], world_size=world, rank=rank, nccl_uid=uid)
        mid = ctx.model_create(shape.dim, shape.heads, shape.ffn, shape.layers, shape.weight_seed)
        for mode in (1, 0):
            ctx.set_option("a2a", mode)
            st0 = ctx.stats()
            req = ctx.submit(mid, 416, 240, 5, 50, 1000, [0, 1])
            assert ctx.run_steps([req], [0, 1], 2) == 2
            z = ctx.read_latent(req)
            ctx.release(req)
            st = ctx.stats()
            out[mode] = (z, st["a2a_peer"] - st0["a2a_peer"], st["a2a_plan"] - st0["a2a_plan"])
        ctx.close()
        q.put((rank, {m: (v[0].tobytes(), v[1], v[2]) for m, v in out.items()}, None))
    except Exception as e:  # noqa: BLE001
        import traceback
        q.put((rank, None, f"{e!r}\n{traceback.format_exc()}"))


def main():
    import numpy as np
    import torch
    import torch.multiprocessing as mp
    import paper_2604_04335_b200 as gs
    from synth import models as sm
    ndev = torch.cuda.device_count()
    dev = [0, 1] if ndev > 1 else [0, 0]
    uid = gs.nccl_unique_id()
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    ps = [ctxm.Process(target=worker, args=(r, 2, uid, dev, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(2):
        r, v, err = q.get(timeout=600)
        if err:
            print(f"rank {r} failed: {err}")
            sys.exit(1)
        res[r] = v
    for p in ps:
        p.join()
    # reference: emulated SP = 2 in this process
    shape = sm.WAN_1_3B.with_layers(2)
    ctx = gs.Context(device=0, world_size=2, emulated=True)
    mid = ctx.model_create(shape.dim, shape.heads, shape.ffn, shape.layers, shape.weight_seed)
    req = ctx.submit(mid, 416, 240, 5, 50, 1000, [0, 1])
    ctx.run_steps([req], [0, 1], 2)
    zref = ctx.read_latent(req)
    ctx.close()
    n = zref.shape[0]
    ok = True
    for mode, name in ((1, "peer"), (0, "plans")):
        # each process writes the token range of the shard it owns; the rest stays zero
        z = np.zeros_like(zref)
        for r in range(2):
            zr = np.frombuffer(res[r][mode][0], dtype=np.float32).reshape(zref.shape)
            lo, hi = r * n // 2, (r + 1) * n // 2
            z[lo:hi] = zr[lo:hi]
        same = np.array_equal(z.view(np.uint32), zref.view(np.uint32))
        print(f"{name}: a2a_peer={res[0][mode][1]} a2a_plan={res[0][mode][2]} bit-exact vs emulated: {same}")
        ok &= same
    print("devices", dev, "OK" if ok else "MISMATCH")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
