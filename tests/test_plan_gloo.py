"""N>1 host logic of the SP path on CPU (no GPU): the exchange plans libgs.so computes for the
Ulysses all-to-alls and the resume re-shard (row a17) are executed
(1) for all positions in one process with NCCL's matching rule and (2) by two real processes over
torch.distributed `gloo` (world_size 2), and the resulting buffers are checked against the
layouts include/gs.h defines, re-derived here from the partition readings (readings 9,
10): token shard i of p = [i n // p, (i+1) n // p); every position holds H // p full heads and the
H % p remaining heads are cut into c = p / gcd(H % p, p) query chunks dealt out in order,
(H % p) / gcd per position (balanced work units)."""
import math
import os
import socket

import numpy as np
import pytest

import paper_2604_04335_b200 as gs


def shards(n, p):
    return [(i * n // p, (i + 1) * n // p) for i in range(p)]


class Units:
    """Balanced head partition (reading 9), re-derived independently of plan.cpp; with
    ring > 1 the USP hybrid's: every head cut into `ring` query chunks, unit (h, ci) on
    position (h // (H // u)) * ring + ci, u = p // ring."""

    def __init__(self, H, p, ring=1):
        if ring > 1 and p % ring == 0 and H % (p // ring) == 0:
            hg = H // (p // ring)
            self.Hf, self.R, self.c = 0, H, ring
            self.units = [((h // hg) * ring + ci, h, ci) for h in range(H) for ci in range(ring)]
            self.of = [[u for u in self.units if u[0] == j] for j in range(p)]
            self.chunks = [[] for _ in range(p)] + [[h] for h in range(H)]
            return
        self.Hf, self.R = H // p, H % p
        g = math.gcd(self.R, p) if self.R else p
        self.c = p // g if self.R else 1
        per = self.R // g if self.R else 0
        self.units = [(k // per, p * self.Hf + k // self.c, k % self.c) for k in range(self.R * self.c)]
        self.of = [[u for u in self.units if u[0] == j] for j in range(p)]
        # pack chunks: p full-head chunks, then one chunk per partial head
        self.chunks = [list(range(j * self.Hf, (j + 1) * self.Hf)) for j in range(p)] + \
                      [[p * self.Hf + u] for u in range(self.R)]

    def chunk_rows(self, n, ci):
        return ci * n // self.c, (ci + 1) * n // self.c


# ----------------------------------------------------------------------------- reference layouts
def send_buffer(q, ns, p, i, H, d, ring=1):
    """Pack layout of position i: chunk j = [rows_i][heads of chunk j][d], chunks in order."""
    U = Units(H, p, ring)
    offs = np.cumsum([0] + ns[:-1])
    rows = np.concatenate([q[o + lo:o + hi] for o, n in zip(offs, ns) for lo, hi in [shards(n, p)[i]]])
    return np.concatenate([rows[:, hs, :].ravel() for hs in U.chunks if hs] + [np.zeros(0, q.dtype)])


def recv_layout(x, ns, p, j, H, kind, ring=1):
    """Receive layout at position j: full heads [rows][Hf][d], then per local unit a [rows][d]
    block: all rows (kind 'kv') or the unit's query-chunk rows of every request (kind 'q', also the
    attention-output layout)."""
    U = Units(H, p, ring)
    offs = np.cumsum([0] + ns[:-1])
    parts = [x[:, j * U.Hf:(j + 1) * U.Hf, :].ravel()]
    for _pos, h, ci in U.of[j]:
        if kind == "kv":
            parts.append(x[:, h, :].ravel())
        else:
            parts.append(np.concatenate([x[o + a:o + b, h, :] for o, n in zip(offs, ns)
                                         for a, b in [U.chunk_rows(n, ci)]]).ravel())
    return np.concatenate(parts)


def execute(plans, bufs):
    """Run per-position plans: n-th send of a to b matched with n-th recv of b from a, then copies."""
    P = len(plans)
    for a in range(P):
        for b in range(P):
            if a == b:
                continue
            snd = [x for x in plans[a] if x["op"] == gs.XFER_SEND and x["peer"] == b]
            rcv = [x for x in plans[b] if x["op"] == gs.XFER_RECV and x["peer"] == a]
            assert len(snd) == len(rcv)
            for s, r in zip(snd, rcv):
                assert s["width"] == r["width"] and s["rows"] == r["rows"] == 1
                src = bufs[a][s["src_buf"]]
                bufs[b][r["dst_buf"]][r["dst_off"]:r["dst_off"] + r["width"]] = \
                    src[s["src_off"]:s["src_off"] + s["width"]]
    for a in range(P):
        for x in plans[a]:
            if x["op"] == gs.XFER_COPY:
                copy_block(bufs[a], x)


def copy_block(bufs, x):
    src, dst = bufs[x["src_buf"]], bufs[x["dst_buf"]]
    for r in range(x["rows"]):
        so = x["src_off"] + r * x["src_pitch"]
        do = x["dst_off"] + r * x["dst_pitch"]
        dst[do:do + x["width"]] = src[so:so + x["width"]]


CASES = [
    (1, [256], 6, 4), (2, [4096 // 64], 12, 8), (2, [33, 17, 64], 12, 8), (4, [1001], 40, 4),
    (8, [75600 // 100], 40, 4), (8, [32760 // 40], 12, 8), (8, [7, 300, 13], 12, 4), (4, [3], 6, 2),
    (8, [101, 29], 6, 4), (4, [55, 2, 77], 6, 4), (8, [300], 13, 2), (2, [9, 1], 5, 2),
]


def test_balanced_units_cover_every_head_row_once_and_balance_work():
    for H in range(1, 41):
        for p in (1, 2, 4, 8):
            U = Units(H, p)
            work = [U.Hf * 1.0] * p
            cover = {}
            for pos, h, ci in U.units:
                work[pos] += 1.0 / U.c
                cover[(h, ci)] = cover.get((h, ci), 0) + 1
            assert all(abs(w - H / p) < 1e-12 for w in work), (H, p, work)
            assert len(cover) == U.R * U.c and set(cover.values()) <= {1}


USP_CASES = [(8, [300], 12, 4, 2), (8, [75600 // 100], 40, 4, 2), (8, [7, 300, 13], 12, 4, 4),
             (8, [101, 29], 40, 2, 8), (4, [55, 2, 77], 6, 4, 2), (4, [1001], 40, 4, 4), (2, [33, 17], 12, 8, 2)]


def test_usp_units_cover_every_head_chunk_once_and_balance_work():
    """USP hybrid partition: every (head, query chunk) exactly once, H / u units per position (each a
    1 / ring share of a head), the units of one head on the `ring` positions of its head group."""
    for H in (6, 12, 40):
        for p in (2, 4, 8):
            for ring in (2, 4, 8):
                if ring > p or p % ring or H % (p // ring):
                    continue
                U = Units(H, p, ring)
                assert sorted((h, ci) for _p, h, ci in U.units) == [(h, ci) for h in range(H) for ci in range(ring)]
                assert all(len(U.of[j]) == H // (p // ring) for j in range(p))
                for h in range(H):
                    pos = sorted(pp for pp, hh, _ci in U.units if hh == h)
                    g = pos[0] // ring
                    assert pos == list(range(g * ring, g * ring + ring))


@pytest.mark.parametrize("p,ns,H,d,ring", [c + (1,) for c in CASES] + USP_CASES)
def test_a2a_plans_realise_ulysses_layouts(p, ns, H, d, ring):
    g = np.random.default_rng(p * 1000 + H)
    N = sum(ns)
    q = g.integers(-1000, 1000, (N, H, d)).astype(np.int64)
    o = g.integers(-1000, 1000, (N, H, d)).astype(np.int64)
    offs = np.cumsum([0] + ns[:-1])
    # seq -> head: K / V (kind 0) and Q (kind 2)
    for kind, name in ((0, "kv"), (2, "q")):
        plans = [gs.plan_a2a(kind, p, i, ns, H, d, ring)[0] for i in range(p)]
        bufs = [{gs.BUF_SEND: send_buffer(q, ns, p, i, H, d, ring),
                 gs.BUF_RECV: np.full(recv_layout(q, ns, p, i, H, name, ring).size, -7, np.int64)}
                for i in range(p)]
        execute(plans, bufs)
        for j in range(p):
            np.testing.assert_array_equal(bufs[j][gs.BUF_RECV], recv_layout(q, ns, p, j, H, name, ring),
                                          err_msg=name)
    # head -> seq
    plans, stages = zip(*[gs.plan_a2a(1, p, i, ns, H, d, ring) for i in range(p)])
    bufs = []
    for i in range(p):
        rows_i = sum(hi - lo for n in ns for lo, hi in [shards(n, p)[i]])
        bufs.append({gs.BUF_O: recv_layout(o, ns, p, i, H, "q", ring).copy(),
                     gs.BUF_STAGE: np.full(max(stages[i], 1), -9, np.int64),
                     gs.BUF_ORECV: np.full(rows_i * H * d, -5, np.int64)})
    execute(plans, bufs)
    for i in range(p):
        want = np.concatenate([o[of + lo:of + hi] for of, n in zip(offs, ns)
                               for lo, hi in [shards(n, p)[i]]]).ravel()
        np.testing.assert_array_equal(bufs[i][gs.BUF_ORECV], want)


RESHARD = [([0], [0]), ([0, 1, 2, 3, 4, 5, 6, 7], [0, 1]), ([0, 1, 2, 3], [4, 5, 6, 7]),
           ([0, 1], [2, 3, 4, 5]), ([4, 5, 6, 7], [0, 1, 2, 3, 4, 5, 6, 7]), ([1, 0], [0, 1]),
           ([3], [0, 1, 2, 3]), ([6, 7], [6])]


@pytest.mark.parametrize("old,new", RESHARD)
@pytest.mark.parametrize("n", [75600 // 50, 1001, 5])
def test_reshard_plans_move_exact_token_ranges(old, new, n):
    lat = 3
    z = np.arange(n * lat, dtype=np.int64)
    plans, bufs = [], []
    for me in range(8):
        plans.append(gs.plan_reshard(n, lat, old, new, me))
        b = {}
        if me in old:
            lo, hi = shards(n, len(old))[old.index(me)]
            b[gs.BUF_OLD] = z[lo * lat:hi * lat].copy()
        if me in new:
            lo, hi = shards(n, len(new))[new.index(me)]
            b[gs.BUF_NEW] = np.full((hi - lo) * lat, -1, np.int64)
        bufs.append(b)
        if me not in old and me not in new:
            assert plans[-1] == []
    execute(plans, bufs)
    for b, me in enumerate(new):
        lo, hi = shards(n, len(new))[b]
        np.testing.assert_array_equal(bufs[me][gs.BUF_NEW], z[lo * lat:hi * lat])


def test_plan_rejects_bad_arguments():
    with pytest.raises(gs.GsError):
        gs.plan_a2a(0, 2, 2, [10], 12, 8)
    with pytest.raises(gs.GsError):
        gs.plan_a2a(5, 2, 0, [10], 12, 8)


# ----------------------------------------------------------------------------- gloo, 2 processes
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run_plan_dist(dist, torch, plan, bufs):
    """Execute one participant's plan over torch.distributed (tag = message index per peer)."""
    reqs, nsent, nrecv = [], {}, {}
    for x in plan:
        if x["op"] == gs.XFER_SEND:
            k = nsent.get(x["peer"], 0)
            nsent[x["peer"]] = k + 1
            t = torch.from_numpy(bufs[x["src_buf"]][x["src_off"]:x["src_off"] + x["width"]].copy())
            reqs.append(dist.isend(t, dst=x["peer"], tag=k))
        elif x["op"] == gs.XFER_RECV:
            k = nrecv.get(x["peer"], 0)
            nrecv[x["peer"]] = k + 1
            t = torch.empty(x["width"], dtype=torch.int64)
            reqs.append((dist.irecv(t, src=x["peer"], tag=k), t, x))
    for r in reqs:
        if isinstance(r, tuple):
            r[0].wait()
            x = r[2]
            bufs[x["dst_buf"]][x["dst_off"]:x["dst_off"] + x["width"]] = r[1].numpy()
        else:
            r.wait()
    for x in plan:
        if x["op"] == gs.XFER_COPY:
            copy_block(bufs, x)


def _worker(rank, world, port, errq):
    try:
        import torch
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        p, ns, H, d = 2, [37, 64, 5], 13, 4  # 13 heads: 6 full each + one head in query halves
        N = sum(ns)
        g = np.random.default_rng(7)      # same seed: every rank knows the global tensors
        q = g.integers(-99, 99, (N, H, d)).astype(np.int64)
        o = g.integers(-99, 99, (N, H, d)).astype(np.int64)
        offs = np.cumsum([0] + ns[:-1])
        me = rank
        for kind, name in ((0, "kv"), (2, "q")):
            plan, _ = gs.plan_a2a(kind, p, me, ns, H, d)
            bufs = {gs.BUF_SEND: send_buffer(q, ns, p, me, H, d),
                    gs.BUF_RECV: np.full(recv_layout(q, ns, p, me, H, name).size, -7, np.int64)}
            _run_plan_dist(dist, torch, plan, bufs)
            np.testing.assert_array_equal(bufs[gs.BUF_RECV], recv_layout(q, ns, p, me, H, name))
        plan, stage = gs.plan_a2a(1, p, me, ns, H, d)
        rows_me = sum(hi - lo for n in ns for lo, hi in [shards(n, p)[me]])
        bufs = {gs.BUF_O: recv_layout(o, ns, p, me, H, "q").copy(),
                gs.BUF_STAGE: np.zeros(max(stage, 1), np.int64),
                gs.BUF_ORECV: np.zeros(rows_me * H * d, np.int64)}
        _run_plan_dist(dist, torch, plan, bufs)
        want = np.concatenate([o[of + lo:of + hi] for of, n in zip(offs, ns)
                               for lo, hi in [shards(n, p)[me]]]).ravel()
        np.testing.assert_array_equal(bufs[gs.BUF_ORECV], want)
        # preempt at SP2 {0,1} -> resume at SP1 {1}, then back to SP2 in swapped order {1,0}
        n, lat = 1001, 4
        z = np.arange(n * lat, dtype=np.int64)
        state = {0: z[:500 * lat].copy(), 1: z[500 * lat:].copy()}[me]
        for old, new in (([0, 1], [1]), ([1], [1, 0]), ([1, 0], [0, 1])):
            plan = gs.plan_reshard(n, lat, old, new, me)
            bufs = {}
            if me in old:
                bufs[gs.BUF_OLD] = state
            if me in new:
                lo, hi = shards(n, len(new))[new.index(me)]
                bufs[gs.BUF_NEW] = np.full((hi - lo) * lat, -1, np.int64)
            _run_plan_dist(dist, torch, plan, bufs)
            state = bufs.get(gs.BUF_NEW)
            if me in new:
                lo, hi = shards(n, len(new))[new.index(me)]
                np.testing.assert_array_equal(state, z[lo * lat:hi * lat])
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        import traceback
        errq.put(f"rank {rank}: {e!r}\n{traceback.format_exc()}")


def test_two_process_gloo_exchange_and_reshard():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, errq)) for r in range(2)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=240)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, "\n".join(errs)
    assert all(pr.exitcode == 0 for pr in procs)


# ----------------------------------------------------------------------------- fused exchange
def peer_stores(q, o, ns, p, me, H, d):
    """Stores position `me` makes under the fused exchange (include/gs.h gs_plan_peer), as
    (destination position, buffer, flat element offsets, values): the pack kernel's Q chunk of
    every destination and its attention output rows scattered to their owners."""
    rd, own_lo, o_base = gs.plan_peer(p, me, ns, H, d)
    Hf, D = H // p, H * d
    offs = np.cumsum([0] + ns[:-1])
    out = []
    # pack: local row m of request r -> full-batch row m + rd[r] of destination j's RECV
    m = 0
    for r, n in enumerate(ns):
        lo, hi = shards(n, p)[me]
        for t in range(lo, hi):
            for j in range(p):
                for hh in range(Hf):
                    base = ((m + rd[r]) * Hf + hh) * d
                    out.append((j, "recv", np.arange(base, base + d), q[offs[r] + t, j * Hf + hh]))
            m += 1
    # attention output of my heads for every row of the batch -> owner's ORECV
    for r, n in enumerate(ns):
        for t in range(n):
            i = max(k for k in range(p) if own_lo[r, k] <= t)
            for hh in range(Hf):
                base = o_base[r, i] + t * D + hh * d
                out.append((i, "orecv", np.arange(base, base + d), o[offs[r] + t, me * Hf + hh]))
    return out


PEER_CASES = [c for c in CASES if c[2] % c[0] == 0] + [(8, [75600 // 100, 37], 40, 2), (2, [1, 1, 3], 2, 3)]


@pytest.mark.parametrize("p,ns,H,d", PEER_CASES)
def test_peer_store_addressing_realises_ulysses_layouts(p, ns, H, d):
    """Fused all-to-alls: the pack kernel's and the attention epilogue's peer stores fill every
    RECV / ORECV element exactly once, with the same bytes the transfer plans deliver."""
    g = np.random.default_rng(p * 77 + H)
    N = sum(ns)
    q = g.integers(-1000, 1000, (N, H, d)).astype(np.int64)
    o = g.integers(-1000, 1000, (N, H, d)).astype(np.int64)
    offs = np.cumsum([0] + ns[:-1])
    rows = [sum(hi - lo for n in ns for lo, hi in [shards(n, p)[i]]) for i in range(p)]
    recv = [np.full(recv_layout(q, ns, p, j, H, "q").size, -7, np.int64) for j in range(p)]
    orecv = [np.full(rows[i] * H * d, -5, np.int64) for i in range(p)]
    hits = [np.zeros(b.size, np.int64) for b in recv], [np.zeros(b.size, np.int64) for b in orecv]
    for me in range(p):
        for dst, buf, idx, val in peer_stores(q, o, ns, p, me, H, d):
            (recv if buf == "recv" else orecv)[dst][idx] = val
            hits[0 if buf == "recv" else 1][dst][idx] += 1
    for j in range(p):
        np.testing.assert_array_equal(recv[j], recv_layout(q, ns, p, j, H, "q"))
        want = np.concatenate([o[of + lo:of + hi] for of, n in zip(offs, ns)
                               for lo, hi in [shards(n, p)[j]]]).ravel()
        np.testing.assert_array_equal(orecv[j], want)
        assert (hits[0][j] == 1).all() and (hits[1][j] == 1).all()


def test_peer_addressing_rejects_uneven_heads():
    with pytest.raises(gs.GsError) as e:
        gs.plan_peer(8, 0, [100], 12, 8)
    assert e.value.code == gs.GS_EUNSUPPORTED
    with pytest.raises(gs.GsError):
        gs.plan_peer(2, 2, [100], 12, 8)


def _peer_worker(rank, world, port, errq):
    """Two processes: each computes its own peer stores and ships them to the destination over
    gloo (standing in for NVLink stores); the receiver's buffers must equal the Ulysses layouts."""
    try:
        import torch
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        p, ns, H, d = 2, [37, 64, 5], 12, 4
        N = sum(ns)
        g = np.random.default_rng(11)
        q = g.integers(-99, 99, (N, H, d)).astype(np.int64)
        o = g.integers(-99, 99, (N, H, d)).astype(np.int64)
        offs = np.cumsum([0] + ns[:-1])
        me = rank
        rows_me = sum(hi - lo for n in ns for lo, hi in [shards(n, p)[me]])
        mine = {"recv": np.full(recv_layout(q, ns, p, me, H, "q").size, -7, np.int64),
                "orecv": np.full(rows_me * H * d, -5, np.int64)}
        outgoing = {"recv": ([], []), "orecv": ([], [])}
        for dst, buf, idx, val in peer_stores(q, o, ns, p, me, H, d):
            if dst == me:
                mine[buf][idx] = val
            else:
                outgoing[buf][0].append(idx)
                outgoing[buf][1].append(val)
        for k, buf in enumerate(("recv", "orecv")):
            idx = np.concatenate(outgoing[buf][0])
            val = np.concatenate(outgoing[buf][1])
            cnt = torch.tensor([idx.size])
            peer_cnt = torch.zeros(1, dtype=torch.int64)
            reqs = [dist.isend(cnt, dst=1 - me, tag=10 + k), dist.irecv(peer_cnt, src=1 - me, tag=10 + k)]
            for r in reqs:
                r.wait()
            pi = torch.empty(int(peer_cnt), dtype=torch.int64)
            pv = torch.empty(int(peer_cnt), dtype=torch.int64)
            reqs = [dist.isend(torch.from_numpy(idx), dst=1 - me, tag=20 + k),
                    dist.isend(torch.from_numpy(val), dst=1 - me, tag=30 + k),
                    dist.irecv(pi, src=1 - me, tag=20 + k), dist.irecv(pv, src=1 - me, tag=30 + k)]
            for r in reqs:
                r.wait()
            mine[buf][pi.numpy()] = pv.numpy()
        np.testing.assert_array_equal(mine["recv"], recv_layout(q, ns, p, me, H, "q"))
        want = np.concatenate([o[of + lo:of + hi] for of, n in zip(offs, ns)
                               for lo, hi in [shards(n, p)[me]]]).ravel()
        np.testing.assert_array_equal(mine["orecv"], want)
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        import traceback
        errq.put(f"rank {rank}: {e!r}\n{traceback.format_exc()}")


def test_two_process_gloo_peer_store_exchange():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_worker, args=(r, 2, port, errq)) for r in range(2)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=240)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, "\n".join(errs)
    assert all(pr.exitcode == 0 for pr in procs)
