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
def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


_ORACLE_BLOCK = {}


def oracle_sample(workload, rows=32):
    """Time the fp64 oracle (oracle/dit.py, as it stands) on SURVEY.md §8(d)'s bounded sample of the
    workload: the row-sampled block of §8(c) "Large configs" on the workload's FULL token grid --
    LN1 and the K/V projections for all n tokens of the (first) request, then the rest of the block
    (q, RMSNorm, RoPE, attention over all n keys, O-proj, MLP) for `rows` seed-chosen query rows
    (first, last and evenly spread rows).  Returns (seconds as run, info); `info` also carries the
    full-step time extrapolated from the measured fp64 rate (labelled as such)."""
    from oracle import dit
    shape, reqs, _ = WORKLOADS[workload]
    w, h, f = reqs[0]
    grid = sm.token_grid(w, h, f)
    n = grid[0] * grid[1] * grid[2]
    if _ORACLE_BLOCK.get(shape.name) is None:  # generated once per process (not timed)
        _ORACLE_BLOCK[shape.name] = sm.as_f64(sm.block_params(shape, 0))
    blk = _ORACLE_BLOCK[shape.name]
    g = np.random.default_rng(5)
    x = g.standard_normal((n, shape.dim))
    e = g.uniform(-0.5, 0.5, (6, shape.dim))
    sel = np.unique(np.concatenate([[0, n - 1], np.linspace(0, n - 1, rows - 2).astype(int)]))
    ctx = g.standard_normal((shape.text_len, shape.dim)) if shape.cross_attn else None
    t0 = time.perf_counter()
    dit.dit_block_rows(x, blk, e, grid, shape.heads, sel, ctx)
    t = time.perf_counter() - t0
    D, F = shape.dim, shape.ffn
    f_kv = 2 * n * 2 * D * D                                 # K and V projections of all tokens
    f_rows = len(sel) * (2 * D * D + 4 * n * D + 2 * D * D + 4 * D * F)   # q, attention, O, MLP
    f_sample = f_kv + f_rows
    full_n = [int(np.prod(sm.token_grid(*r))) for r in reqs]
    nb = 2 if CFG_SCALE.get(workload, 0.0) > 0 else 1
    f_block = costmodel.flops_per_block(full_n, D, F)
    if shape.cross_attn:
        f_block += sum(4 * m * D * D + 4 * m * shape.text_len * D for m in full_n)
    f_step = nb * shape.layers * f_block
    rate = f_sample / t
    info = {"sample": (f"oracle dit_block_rows (fp64 numpy, as run) of layer 0 of {shape.name} on the "
                       f"full {grid} grid ({n} tokens): LN1 + K/V projections of all tokens + the rest "
                       f"of the block for {len(sel)} sampled query rows ({f_sample / 1e12:.2f} TFLOP)"),
            "sample_s": round(t, 3), "gflops_fp64": round(rate / 1e9, 2),
            "extrapolated_full_step_ms": round(f_step / rate * 1e3, 1),
            "extrapolation": (f"full {shape.layers}-layer step = {f_step / 1e12:.1f} TFLOP at the "
                              "measured fp64 rate (labelled extrapolation, not a measurement)")}
    return t, info


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def run_reference(args, rank, world):
    """--impl reference: the oracle on the host cores, rank 0 only (other ranks exit 0).  Each
    step is the bounded sample of oracle_sample() (the same quantity as the GPU arm's
    cpu_baseline), timed as run: `value` is the measured ms of one sample, so
    value x steps fits inside the run's own wall clock."""
    if rank != 0:
        return
    times, info = [], None
    for i in range(args.warmup + args.steps):
        t, info = oracle_sample(args.workload)
        if i >= args.warmup:
            times.append(t * 1e3)
    v = float(np.mean(times))
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 1), "unit": "ms",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(v, 1), "higher_is_better": False,
            "scaling": "strong" if WORKLOADS[args.workload][2] else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded splitmix64)",
            "config": {"workload": CONFIG_NAME[args.workload], "sp": 1,
                       "step": "one bounded oracle sample (see cpu_baseline.sample)"},
            "cpu_baseline": {"value": round(v, 1), "unit": "ms", "cores": host_cores(), "kind": "oracle",
                             "cpu_model": cpu_model(), "sample": info["sample"],
                             "gflops_fp64": info["gflops_fp64"],
                             "extrapolated_full_step_ms": info["extrapolated_full_step_ms"],
                             "extrapolation": info["extrapolation"]},
            "e2e": {"value": round(v, 1), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
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


def kernel_class_rates(st, steps, shape, rows_per_pos, seqlens, heads_local, nb=1):
    """Attention and GEMM TFLOP/s of the profiled steps from gs_stats per-class events."""
    attn = st.get("attention", {"ms": 0.0, "n": 0})
    gemm_ms = sum(v["ms"] for k, v in st.items() if isinstance(v, dict) and k.startswith("gemm"))
    gemm_n = sum(v["n"] for k, v in st.items() if isinstance(v, dict) and k.startswith("gemm"))
    af = attn_flops_per_launch(shape, list(seqlens) * nb, heads_local)
    attn_avg = attn["ms"] / max(attn["n"], 1)
    gf = shape.layers * costmodel.gemm_flops_per_block(rows_per_pos, shape.dim, shape.ffn)
    return {"attn_tflops": round(af / (attn_avg * 1e-3) / 1e12, 1) if attn_avg > 0 else None,
            "attn_ms_per_step": round(attn["ms"] / steps, 3),
            "attn_launch_ms": round(attn_avg, 4),
            "gemm_ms_per_step": round(gemm_ms / steps, 3),
            "gemm_launches_per_step": gemm_n // max(steps, 1),
            "gemm_flops_per_position_step": gf}


def t2i_secondary(gs, torch, pk, steps=40, warmup=3):
    """The T2I half of the headline metric (BASELINE.json: "... 720p T2V + 1024px T2I"): config 2,
    4 x 1024^2 images batched on one GPU (Wan-1.3B-shaped, L = 30), device-timed steps with the
    clocks sampled through a ~2 s timed region (>= 10 samples), then one per-kernel-profiled step."""
    shape, reqs_spec, _ = WORKLOADS["t2i1024"]
    ctx = gs.Context(device=0)
    mid = ctx.model_create(shape.dim, shape.heads, shape.ffn, shape.layers, shape.weight_seed)
    reqs = [ctx.submit(mid, w, h, f, 100, 1000 + r, [0]) for r, (w, h, f) in enumerate(reqs_spec)]
    ctx.run_steps(reqs, [0], warmup)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr(0))
    ctx.profile(2, True)
    clocks = ClockSampler(0)
    clocks.start()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks.mark_start()
    e0.record(stream)
    ctx.run_steps(reqs, [0], steps)
    e1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / steps
    step_ms = ctx.stats().get("step_ms", [])
    ctx.profile(1, True)
    ctx.run_steps(reqs, [0], 2)
    st = ctx.stats()
    ctx.profile(0, False)
    ctx.close()
    seqlens = [int(np.prod(sm.token_grid(*r))) for r in reqs_spec]
    rates = kernel_class_rates(st, 2, shape, sum(seqlens), seqlens, shape.heads)
    gt = rates["gemm_flops_per_position_step"] / (rates["gemm_ms_per_step"] * 1e-3) / 1e12
    return {"workload": CONFIG_NAME["t2i1024"], "ms_per_step": round(ms, 3), "steps": steps,
            "warmup": warmup, "step_cv": round(float(np.std(step_ms) / np.mean(step_ms)), 5),
            "attn_tflops": rates["attn_tflops"],
            "attn_frac_sustained": round(rates["attn_tflops"] / pk["bf16_sustained"], 4),
            "gemm_tflops": round(gt, 1), "gemm_frac_sustained": round(gt / pk["bf16_sustained"], 4),
            "attn_ms_per_step": rates["attn_ms_per_step"], "gemm_ms_per_step": rates["gemm_ms_per_step"],
            "clocks": clk}


def vae_decode_720p(gs, torch, pk, reps=2):
    """NEXT-4: the VAE decode stage of config 4's request on ONE GPU (the VAE stage always
    runs on a single GPU, decoupled from the DiT): a 720x1280 / 81-frame latent (DiT grid 21 x 45 x 80)
    through the Wan2.1-VAE-shaped decoder to 81 x 720 x 1280 x 3, inputs and outputs
    resident on the device; device-timed with CUDA events.  TFLOP/s counts the algorithmic conv work
    (unpadded channels; costmodel.vae_decode_flops).  Paper context (Tab. stage_breakdown):
    2.47 s VAE decode at 720p for Wan2.2-5B on its own GPU -- another VAE and GPU."""
    grid = (21, 45, 80)
    ctx = gs.Context(device=0)
    vid = ctx.vae_create()
    lat = torch.randn(int(np.prod(grid)) * 64, device="cuda", dtype=torch.float32)
    shape = ctx.vae_out_shape(grid)
    out = torch.empty(shape, device="cuda", dtype=torch.float32)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr(0))
    ctx.vae_decode(vid, lat, grid, out=out)          # warm-up (first-use allocations)
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ctx.vae_decode(vid, lat, grid, out=out)
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ok = bool(torch.isfinite(out).all().item()) and float(out.abs().max().item()) <= 1.0
    ctx.close()
    ms = float(np.median(ts))
    fl = costmodel.vae_decode_flops(grid)
    tf = fl / (ms * 1e-3) / 1e12
    return {"workload": "Wan2.1-VAE-shaped decode of config 4's latent: 21x90x160x16 -> 81x720x1280x3, 1 GPU",
            "ms": round(ms, 2), "reps": reps, "tflops_algorithmic": round(tf, 1),
            "frac_sustained": round(tf / pk["bf16_sustained"], 4), "flops": fl,
            "output_in_range": ok,
            "note": "activation buffers grow once and are re-used; channels padded to multiples of 32 (the "
                    "96-channel last stage runs unpadded on 32-channel K blocks); conv work runs on tcgen05 "
                    "implicit-GEMM kernels, norms / upsampling on HBM-bound kernels",
            "paper_context": "Tab. stage_breakdown: VAE Dec. 2.47 s at 720p/81f (Wan2.2-5B, RTX PRO 6000)"}


def sp8_emulated(gs, torch, pk):
    """Config 4 at the north-star shape on one GPU: the 720p/81f Wan-14B-shaped request at SP = 8 in
    the emulated context (8 virtual ranks, each position = 9,450 rows and 5 of the 40 heads; the
    positions run one after another on this GPU and the all-to-alls are device copies), so the
    per-position kernels run at exactly the per-GPU shape of an 8-GPU run.  Reports the step time
    (all 8 positions), the per-position attention / GEMM rates and fractions of the step, then
    config 4's preempt -> re-shard -> resume at SP = 2 on GPUs {0, 1}: the gs_preempt call, the
    wait until the in-flight step's boundary, and the SP8 -> SP2 re-shard (gs_resume) with the
    bytes the plan moves (PAPER.md Tab. preemption_scaling P:794-797 is context: other GPUs, PCIe)."""
    shape = sm.WAN_14B
    p, n = 8, int(np.prod(sm.token_grid(1280, 720, 81)))
    ctx = gs.Context(device=0, world_size=8, emulated=True)
    mid = ctx.model_create(shape.dim, shape.heads, shape.ffn, shape.layers, shape.weight_seed)
    ranks = list(range(p))
    req = ctx.submit(mid, 1280, 720, 81, 50, 1000, ranks)
    ctx.run_steps([req], ranks, 1)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr(0))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    ctx.run_steps([req], ranks, 1)
    e1.record(stream)
    torch.cuda.synchronize()
    step_ms = e0.elapsed_time(e1)
    ctx.profile(1, True)
    ctx.run_steps([req], ranks, 1)
    st = ctx.stats()
    ctx.profile(0, False)
    rates = kernel_class_rates(st, 1, shape, n // p, [n], shape.heads // p)
    gt = rates["gemm_flops_per_position_step"] * p / (rates["gemm_ms_per_step"] * 1e-3) / 1e12
    a2a_ms = sum(v["ms"] for k, v in st.items() if isinstance(v, dict) and k.startswith("a2a"))
    # preempt a run in flight: the call itself, then the wait for the step boundary
    t = ctx.run_steps_async([req], ranks, 2)
    time.sleep(0.5)
    c0 = time.perf_counter()
    ctx.preempt(req)
    c1 = time.perf_counter()
    ran = ctx.wait(t)
    c2 = time.perf_counter()
    assert ctx.query(req)["state"] == gs.REQ_PAUSED
    calls = []
    for _ in range(200):  # the call on a paused request (flag + state under the table lock)
        a = time.perf_counter()
        ctx.preempt(req)
        calls.append(time.perf_counter() - a)
    plan_bytes, into_one = 0, 0
    for me in range(8):
        xs = gs.plan_reshard(n, 64, ranks, [0, 1], me)
        plan_bytes += sum(x["width"] * 4 for x in xs if x["op"] == gs.XFER_SEND)
        into_one = max(into_one, sum(x["width"] * 4 for x in xs if x["op"] == gs.XFER_RECV))
    torch.cuda.synchronize()
    r0 = time.perf_counter()
    ctx.resume(req, [0, 1])
    r1 = time.perf_counter()
    ok = ctx.run_steps([req], [0, 1], 1) == 1
    ctx.close()
    return {"workload": "config4 720x1280 81f Wan-14B-shaped at SP=8, emulated on 1 GPU "
                        "(per-position shapes of the 8-GPU run; exchanges as device copies)",
            "step_ms_all_positions": round(step_ms, 2),
            "position_step_ms_est": round(step_ms / p, 2),
            "attn_tflops_per_launch": rates["attn_tflops"],
            "attn_frac_sustained": round(rates["attn_tflops"] / pk["bf16_sustained"], 4),
            "attn_frac_of_step": round(rates["attn_ms_per_step"] / step_ms, 4),
            "gemm_tflops": round(gt, 1), "gemm_frac_sustained": round(gt / pk["bf16_sustained"], 4),
            "gemm_frac_of_step": round(rates["gemm_ms_per_step"] / step_ms, 4),
            "a2a_copy_ms_per_step": round(a2a_ms, 3),
            "preempt": {"call_us_in_flight": round((c1 - c0) * 1e6, 1),
                        "call_us_median": round(float(np.median(calls)) * 1e6, 2),
                        "until_step_boundary_ms": round((c2 - c1) * 1e3, 1), "steps_run_before_pause": ran,
                        "paper_context": "Tab. preemption_scaling: pause 3.0-3.4 us (P:794-797)"},
            "resume_sp8_to_sp2": {"ms": round((r1 - r0) * 1e3, 3), "bytes_moved": plan_bytes,
                                  "max_bytes_into_one_gpu": into_one, "run_after_ok": ok,
                                  "nvlink_lower_bound_us": round(into_one / 900e9 * 1e6, 1),
                                  "how": "gs_resume wall clock (plan + device copies on one GPU, synchronised)",
                                  "paper_context": "Tab. preemption_scaling: resume 0.036-0.868 ms (P:794-797)"}}


def run_gpu(args, rank, world, local_rank):
    import torch
    import paper_2604_04335_b200 as gs

    dist = None
    if world > 1:
        # NCCL's INIT lines (stderr) show each rank's communicator and nranks for the driver's log
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        uid = [gs.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx = gs.Context(device=local_rank, world_size=world, rank=rank, nccl_uid=uid[0])
        inf = ctx.info()
        print(f"[bench] rank {rank}/{world}: gs context on cuda:{local_rank}, NCCL world {inf['world_size']}, "
              f"{inf['num_sms']} SMs", file=sys.stderr, flush=True)
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
            # q, k bf16 in, normalised / rotated q, k out; v is moved too (packed for the exchange) only at SP > 1
            # -- at SP = 1 the attention reads V in place from the QKV GEMM output
            "qk_norm_rope": ("hbm", rows * (2 if p == 1 else 3) * D * 2 * 2)}
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

    extra = {}
    if world == 1 and not args.no_secondary:
        ctx.close()
        ctx = None
        torch.cuda.empty_cache()
        extra["t2i1024"] = t2i_secondary(gs, torch, pk)
        extra["sp8_emulated"] = sp8_emulated(gs, torch, pk)
        extra["vae_decode_720p"] = vae_decode_720p(gs, torch, pk)

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        t_cpu, info = oracle_sample(args.workload)
        cpu = {"value": round(t_cpu * 1e3, 1), "unit": "ms", "cores": host_cores(), "kind": "oracle",
               "cpu_model": cpu_model(), "sample": info["sample"], "gflops_fp64": info["gflops_fp64"],
               "extrapolated_full_step_ms": info["extrapolated_full_step_ms"],
               "extrapolation": info["extrapolation"]}

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
                     "frac_of_datasheet": round(achieved / 2250.0, 4),
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
        "step_cv_context": "paper Tab. 1 (P:170-173, SURVEY §8(c) P7): per-step latency CV <= 0.04% on its GPUs; "
                           "ours includes the power-capped clock wander of this box (clocks.reasons)",
        "gpu_launches": int(launches),
        "e2e": {"value": round(e2e_v, 3), "unit": "ms", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": lat_bytes, "steps": e2e_steps,
                "how": "wall clock around gs_submit(pinned host latent) + gs_run_steps(k=1) + "
                       "gs_read_latent(into pinned host buffers) + gs_release"},
        "clocks": clk,
        "cpu_baseline": cpu,
    }
    line.update(extra)
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    if ctx is not None:
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
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the N=1 secondary objects (t2i1024, sp8_emulated with preempt/resume)")
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
