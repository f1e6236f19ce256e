"""bench.py — DiT denoising-step benchmark of the GenServe hot path on B200.

Contract (task statement / DESIGN.md "Measurement"):
  python bench.py --gpus N --steps K --warmup W [--workload W] [--impl reference]
prints ONE JSON line on rank 0.  Under torchrun (N > 1) every rank owns one GPU; the request is
token-sharded over all N ranks (Ulysses SP degree p = N) and the exchanges run over NCCL.

A "step" is one whole pass of the hot path: time embedding, patch
embed, L DiT blocks (LN+mod, QKV GEMM, qk-RMSNorm+RoPE+pack, a2a, flash attention, a2a, O GEMM +
gated residual, LN+mod, MLP up+GELU, MLP down + gated residual), head + Euler update, for one
batch of synthetic input.  Workloads (BASELINE.json configs):
  t2v720  (default) config 4: 720x1280, 81 frames -> 75,600 tokens, Wan-14B-shaped (D 5120,
          40x128 heads, F 13824, L 40), one request at SP = N  ("scaling": "strong")
  t2v480  config 3: 480x832, 81 frames -> 32,760 tokens, Wan-1.3B-shaped, SP = N (strong)
  t2i1024 config 2: 4 x 1024^2 images (4 x 4096 tokens), Wan-1.3B-shaped, SP = 1 per rank;
          N > 1 runs N independent image batches (replicas, "scaling": "weak")
The metric is BASELINE.json's "DiT step ms & attn TFLOPS (% BF16 peak)": `value` is the DiT
step time (ms, device-timed with CUDA events on the context's stream, max over ranks; the timed
steps carry only per-step events, whose spread gives `step_cv`); attention TFLOPS and its fraction
of the measured BF16 peak ride in `roofline`, from per-kernel events of --prof-steps extra steps
run after the timed region.
Inputs are far larger than L2 (weights 19.7 GB / 2.6 GB, activations > 1 GB), so no explicit
L2 flush is needed between timed steps ("l2": "inputs larger than L2" in config).

`--impl reference` is the base contract's reference arm for this tier: the fp64 CPU oracle
(oracle/dit.py) timed as it stands on the host cores on a bounded sample of the same workload.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2604_04335_b200 import costmodel  # noqa: E402  (work accounting, no method arithmetic)
from synth import models as sm  # noqa: E402

METRIC = "DiT step ms & attn TFLOPS (% BF16 peak) at SP=1/2/4/8, 720p T2V + 1024px T2I"

WORKLOADS = {
    # name: (model shape, [(width, height, frames)], sp_over_ranks)
    "t2v720": (sm.WAN_14B, [(1280, 720, 81)], True),
    "t2v480": (sm.WAN_1_3B, [(832, 480, 81)], True),
    "t2i1024": (sm.WAN_1_3B, [(1024, 1024, 1)] * 4, False),
    # NEXT-1: the full Wan block (text cross-attention over 512 prompt tokens) with classifier-free
    # guidance g = 5 (cond + uncond forward per step)
    "t2v720_text_cfg": (sm.WAN_14B.with_text(512, 4096), [(1280, 720, 81)], True),
}
CFG_SCALE = {"t2v720_text_cfg": 5.0}
CONFIG_NAME = {
    "t2v720": "config4: 720x1280 81f T2V (75600 tok), Wan-14B-shaped DiT step",
    "t2v480": "config3: 480x832 81f T2V (32760 tok), Wan-1.3B-shaped DiT step",
    "t2i1024": "config2: 4 x 1024px T2I (4 x 4096 tok) batch, Wan-1.3B-shaped DiT step",
    "t2v720_text_cfg": "config4 + NEXT-1: 720x1280 81f T2V, Wan-14B-shaped step with text "
                       "cross-attention (512 tok) and CFG g=5 (2 forwards)",
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return {"hbm": p["hbm_gbs"], "bf16": p["bf16_tflops"],
                "bf16_sustained": p["bf16_tflops_sustained"], "src": "measured"}
    except Exception:
        # /opt/skills/guides/B200_PROFILING.md fallback figures
        return {"hbm": 6650.0, "bf16": 1590.0, "bf16_sustained": 1400.0, "src": "fallback"}


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region (B200_PROFILING.md)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    REASONS = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.mark = 0

    def start(self):
        """Start sampling (every 100 ms) and wait for the first sample, so that a short timed
        region (a config-2 step is ~50 ms) still has samples; call mark() where it begins."""
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 10:
                time.sleep(0.01)
        except Exception:
            self.proc = None

    def mark_start(self):
        self.mark = len(self.lines)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        # samples taken inside the timed region; if it was shorter than the sampling interval, the
        # samples nearest to it (the last one before and the first one after)
        inside = self.lines[self.mark:]
        near = inside if inside else self.lines[max(self.mark - 1, 0):self.mark + 1]
        sms, maxs, pw, reasons = [], [], [], set()
        for ln in near:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sms.append(float(f[1]))
                maxs.append(float(f[2]))
            except ValueError:
                continue
            try:
                pw.append(float(f[3]))
            except ValueError:
                pass
            for name, v in zip(self.REASONS, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        if not sms:
            return None
        return {"sm_mhz": float(np.median(sms)), "sm_max_mhz": max(maxs),
                "power_w": float(np.median(pw)) if pw else None,
                "reasons": sorted(reasons), "samples": len(sms), "in_region": bool(inside)}


# ----------------------------------------------------------------------------- oracle sample
def oracle_sample(workload, reps=1, budget_tokens=None):
    """Time the fp64 oracle (as it stands) on a bounded sample of the workload: one full DiT
    block of layer 0 on a single-latent-frame request of the workload's resolution (fewer
    tokens, same model dims), then extrapolate to one full step by the paper's FLOP model
    (PAPER.md Tab. arithmetic_intensity; costmodel.py).  Returns (ms_per_full_step, info)."""
    from oracle import dit
    shape, reqs, _ = WORKLOADS[workload]
    w, h, _f = reqs[0]
    grid = sm.token_grid(w, h, 1)
    if budget_tokens is not None and grid[1] * grid[2] > budget_tokens:
        rows = max(1, budget_tokens // grid[2])
        grid = (1, rows, grid[2])
    n = grid[0] * grid[1] * grid[2]
    blk = sm.as_f64(sm.block_params(shape, 0))
    g = np.random.default_rng(5)
    x = g.standard_normal((n, shape.dim))
    e_req = g.uniform(-0.5, 0.5, (1, 6, shape.dim))
    ctxs = [g.standard_normal((shape.text_len, shape.dim))] if shape.cross_attn else None
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        dit.dit_block(x, blk, e_req, [(0, n, grid)], shape.heads, ctxs)
        times.append(time.perf_counter() - t0)
    t = float(np.median(times))

    def block_flops(ns):
        f = costmodel.flops_per_block(ns, shape.dim, shape.ffn)
        if shape.cross_attn:  # cross q/o projections + attention over the text tokens
            f += sum(4 * m * shape.dim ** 2 + 4 * m * shape.text_len * shape.dim for m in ns)
        return f
    f_sample = block_flops([n])
    full_seqs = [sm.token_grid(*r) for r in reqs]
    full_n = [a * b * c for a, b, c in full_seqs]
    nb = 2 if CFG_SCALE.get(workload, 0.0) > 0 else 1
    f_step = nb * shape.layers * block_flops(full_n)
    ms_step = t * 1e3 * f_step / f_sample
    info = {"sample": (f"oracle dit_block (fp64 numpy) layer 0 of {shape.name} on a {grid} "
                       f"token grid ({n} tokens, {f_sample / 1e9:.1f} GFLOP) in {t:.2f} s; "
                       f"extrapolated by FLOPs to one full {shape.layers}-layer step of "
                       f"{sum(full_n)} tokens ({f_step / 1e12:.1f} TFLOP)"),
            "sample_s": t, "gflops_fp64": f_sample / t / 1e9}
    return ms_step, info


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def run_reference(args, rank, world):
    """--impl reference: the oracle on the host cores, rank 0 only."""
    if rank != 0:
        return
    times, info = [], None
    for i in range(args.warmup + args.steps):
        ms, info = oracle_sample(args.workload, reps=1, budget_tokens=args.ref_tokens)
        if i >= args.warmup:
            times.append(ms)
    v = float(np.mean(times))
    shape, reqs, _ = WORKLOADS[args.workload]
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "ms",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": v, "higher_is_better": False,
            "scaling": "strong" if WORKLOADS[args.workload][2] else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded splitmix64)",
            "config": {"workload": CONFIG_NAME[args.workload], "sp": 1},
            "cpu_baseline": {"value": v, "unit": "ms", "cores": host_cores(), "kind": "oracle",
                             "sample": info["sample"]},
            "e2e": {"value": v, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm
def attn_flops_per_launch(shape, seqlens, heads_local):
    return 4 * shape.head_dim * heads_local * sum(n * n for n in seqlens)


def head_split(H, p, j):
    return (j + 1) * (H // p) + min(j + 1, H % p) - (j * (H // p) + min(j, H % p))


def load_traffic(workload, p):
    """dram bytes per attention launch from a committed ncu --set full capture, if any."""
    path = os.path.join(ROOT, "profiles", "attention_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(f"{workload}_sp{p}")
    except Exception:
        return None


def run_gpu(args, rank, world, local_rank):
    import torch
    import paper_2604_04335_b200 as gs

    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        uid = [gs.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx = gs.Context(device=local_rank, world_size=world, rank=rank, nccl_uid=uid[0])
    else:
        torch.cuda.set_device(local_rank)
        ctx = gs.Context(device=local_rank)

    shape, reqs_spec, sp_over_ranks = WORKLOADS[args.workload]
    ranks = list(range(world)) if sp_over_ranks else [rank]
    p = len(ranks)
    if not sp_over_ranks and world > 1:
        # replicas: every rank owns its own single-rank placement (images use <= 1 GPU)
        pass
    mid = ctx.model_create(shape.dim, shape.heads, shape.ffn, shape.layers, shape.weight_seed,
                           cross_attn=shape.cross_attn, text_len=shape.text_len, text_dim=shape.text_dim)
    total_steps = max(50, args.warmup + args.steps + args.prof_steps + 1)
    cfg = CFG_SCALE.get(args.workload, 0.0)
    nb = 2 if cfg > 0 else 1

    def submit_all(init=None):
        out = []
        for r, (w, h, f) in enumerate(reqs_spec):
            lat = None if init is None else init[r]
            if shape.cross_attn:
                out.append(ctx.submit_text(mid, w, h, f, total_steps, 1000 + r, ranks, prompt_seed=2000 + r,
                                           cfg_scale=cfg, init_latent=lat))
            else:
                out.append(ctx.submit(mid, w, h, f, total_steps, 1000 + r, ranks, init_latent=lat))
        return out

    stream = torch.cuda.ExternalStream(ctx.stream_ptr(rank))

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if dist is None:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # -------------------------------------------------------------- device-timed steps
    reqs = submit_all()
    if args.warmup:
        ctx.run_steps(reqs, ranks, args.warmup)
    ctx.profile(2, True)  # step events only: the timed steps carry no per-kernel events
    clocks = ClockSampler(local_rank) if rank == 0 else None
    if clocks:
        clocks.start()  # before the barrier: waiting for its first sample must not skew the ranks
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    if clocks:
        clocks.mark_start()
    ev0.record(stream)
    done = ctx.run_steps(reqs, ranks, args.steps)
    ev1.record(stream)
    barrier()
    clk = clocks.stop() if clocks else None
    assert done == args.steps, f"ran {done} of {args.steps} steps"
    ms_total = max_over_ranks(ev0.elapsed_time(ev1))
    ms_step = ms_total / args.steps
    step_ms = ctx.stats().get("step_ms", [])
    launches = ctx.stats().get("launches", 0)
    # per-kernel-class breakdown (attention / GEMM TFLOP/s, roofline) from separate profiled
    # steps, so the per-kernel events never sit inside the timed region
    ctx.profile(1, True)
    ctx.run_steps(reqs, ranks, args.prof_steps)
    st = ctx.stats()
    ctx.profile(0, False)
    for q in reqs:
        ctx.release(q)

    # -------------------------------------------------------------- end to end (host buffers)
    seqlens = [int(np.prod(sm.token_grid(*r))) for r in reqs_spec]

    def pinned(n):  # page-locked host buffer (numpy view of a pinned torch tensor)
        return torch.empty((n, 64), dtype=torch.float32, pin_memory=True).numpy()

    host_z = []
    for i, n in enumerate(seqlens):
        z = pinned(n)
        z[...] = np.random.default_rng(40 + i).standard_normal((n, 64))
        host_z.append(z)
    host_out = [pinned(n) for n in seqlens]
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    e2e_ms = []
    out = None
    for _ in range(e2e_steps):
        barrier()
        t0 = time.perf_counter()
        rq = submit_all(host_z)                       # H2D of the step's input latents
        ctx.run_steps(rq, ranks, 1)
        out = [ctx.read_latent(q, n, out=o) for q, n, o in zip(rq, seqlens, host_out)]   # D2H of the result
        for q in rq:
            ctx.release(q)
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2e_v = max_over_ranks(float(np.median(e2e_ms)))
    lat_bytes = sum(seqlens) * 64 * 4
    # each rank copies its own shard in and out
    h2d = lat_bytes if not sp_over_ranks else lat_bytes  # whole-job bytes per step
    assert out is not None and all(np.isfinite(o).all() for o in out)

    if rank != 0:
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        ctx.close()
        return

    # -------------------------------------------------------------- roofline (attention)
    pk = peaks()
    H_loc = head_split(shape.heads, p, 0)  # rank 0 carries the most heads
    attn = st.get("attention", {"ms": 0.0, "n": 0})
    attn_avg_ms = attn["ms"] / max(attn["n"], 1)
    af = attn_flops_per_launch(shape, seqlens * nb, H_loc)  # CFG: cond + uncond sequences
    achieved = af / (attn_avg_ms * 1e-3) / 1e12 if attn_avg_ms > 0 else 0.0
    peak = pk["bf16_sustained"]
    traffic = load_traffic(args.workload, p)
    gemm_ms = sum(v["ms"] for k, v in st.items() if isinstance(v, dict) and k.startswith("gemm"))
    rows = nb * sum(seqlens) / p
    cross_gemm = 4 * rows * shape.dim ** 2 if shape.cross_attn else 0  # cross q and o projections
    gemm_flops = shape.layers * (costmodel.gemm_flops_per_block(rows, shape.dim, shape.ffn) + cross_gemm)
    gemm_tflops = gemm_flops * args.prof_steps / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else 0.0
    cross_attn_flops = 4 * rows * shape.text_len * shape.dim if shape.cross_attn else 0
    step_flops = shape.layers * (costmodel.gemm_flops_per_block(rows, shape.dim, shape.ffn) + cross_gemm + af
                                 + cross_attn_flops)
    breakdown = {k: round(v["ms"] / args.prof_steps, 3) for k, v in st.items() if isinstance(v, dict)}
    # per kernel class: algorithmic work per launch / average launch time vs its roofline
    # (DESIGN.md §6): GEMMs against the bf16 tensor peak, row kernels against HBM bandwidth
    D, F = shape.dim, shape.ffn
    work = {"gemm_qkv": ("tensor", 2 * rows * D * 3 * D), "gemm_o": ("tensor", 2 * rows * D * D),
            "gemm_mlp_up": ("tensor", 2 * rows * D * F), "gemm_mlp_down": ("tensor", 2 * rows * F * D),
            "ln_mod": ("hbm", rows * D * (4 + 2)),            # x fp32 in, a bf16 out
            "qk_norm_rope": ("hbm", rows * 3 * D * 2 * 2)}    # q|k|v bf16 in, packed q, k, v out
    kernels = {}
    for k, (bound, per_launch) in work.items():
        v = st.get(k)
        if not isinstance(v, dict) or v["n"] == 0 or v["ms"] <= 0:
            continue
        avg_s = v["ms"] / v["n"] * 1e-3
        if bound == "tensor":
            ach, unit, pkv = per_launch / avg_s / 1e12, "TFLOP/s", pk["bf16_sustained"]
        else:
            ach, unit, pkv = per_launch / avg_s / 1e9, "GB/s", pk["hbm"]
        kernels[k] = {"bound": bound, "achieved": round(ach, 1), "peak": pkv, "unit": unit,
                      "frac": round(ach / pkv, 4), "avg_launch_us": round(avg_s * 1e6, 1),
                      "peak_src": ("measured bf16 sustained; frac_of_burst vs " + str(pk["bf16"]))
                      if bound == "tensor" else "measured HBM copy bandwidth",
                      "launches_per_step": v["n"] // args.prof_steps,
                      ("flops" if bound == "tensor" else "bytes") + "_per_launch": int(per_launch)}
        if bound == "tensor":
            kernels[k]["frac_of_burst"] = round(ach / pk["bf16"], 4)

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        ms_cpu, info = oracle_sample(args.workload, reps=1, budget_tokens=args.ref_tokens)
        cpu = {"value": ms_cpu, "unit": "ms", "cores": host_cores(), "kind": "oracle",
               "sample": info["sample"], "gflops_fp64": round(info["gflops_fp64"], 2)}

    line = {
        "metric": METRIC, "value": round(ms_step, 3), "unit": "ms", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 3),
        "higher_is_better": False, "scaling": "strong" if sp_over_ranks else "weak",
        "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded splitmix64 latents, random-init weights of the shape)",
        "config": {"workload": CONFIG_NAME[args.workload], "sp": p,
                   "tokens": seqlens, "layers": shape.layers, "dim": shape.dim,
                   "heads": shape.heads, "ffn": shape.ffn,
                   "parallelism": f"ulysses_sp{p}" if sp_over_ranks else f"replicas{world}",
                   "l2": "inputs larger than L2 (no flush)"},
        "roofline": {"bound": "tensor", "kernel": "attention (attn_tc_kernel<128>)",
                     "achieved": round(achieved, 1), "peak": peak, "unit": "TFLOP/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic,
                     "peak_src": f"{pk['src']} bf16 sustained (kernel timed inside a long step)",
                     "frac_of_burst": round(achieved / pk["bf16"], 4),
                     "flops_per_launch": af, "avg_launch_ms": round(attn_avg_ms, 4),
                     "algorithmic_bytes_per_launch": 4 * sum(seqlens) * H_loc * shape.head_dim * 2,
                     "traffic_src": "profiles/attention_traffic.json (ncu --set full, dram read+write "
                                    "per launch at this shape)"},
        "attn_tflops": round(achieved, 1),
        "gemm_tflops": round(gemm_tflops, 1),
        "step_tflops": round(step_flops / (ms_step * 1e-3) / 1e12, 1),
        "breakdown_ms_per_step": breakdown,
        "breakdown_steps": args.prof_steps,
        "kernels": kernels,
        "step_ms_each": [round(x, 3) for x in step_ms],
        "step_cv": round(float(np.std(step_ms) / np.mean(step_ms)), 5) if len(step_ms) > 1 else None,
        "gpu_launches": int(launches),
        "e2e": {"value": round(e2e_v, 3), "unit": "ms", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": lat_bytes, "steps": e2e_steps,
                "how": "wall clock around gs_submit(pinned host latent) + gs_run_steps(k=1) + "
                       "gs_read_latent(into pinned host buffers) + gs_release"},
        "clocks": clk,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    ctx.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="t2v720", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--prof-steps", type=int, default=2,
                    help="extra per-kernel-profiled steps after the timed region (breakdown, roofline)")
    ap.add_argument("--ref-tokens", type=int, default=1200,
                    help="token budget of the oracle sample (bounded CPU time)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            sys.exit("bench.py --gpus N>1 must be launched under torchrun (one rank per GPU)")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_gpu(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
