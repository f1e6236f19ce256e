"""Kernel micro-benchmarks (development aid, not the bench contract): times the tcgen05 GEMM and
flash-attention kernels through the C-ABI debug entry points at the shapes of BASELINE.json's
configs, with CUDA events on the context's stream, and prints TFLOP/s vs the measured peak.

  python tools/kbench.py [--attn] [--gemm] [--reps 5]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2604_04335_b200 as gs  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"] \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 1590.0

# (label, seqlens, heads, d): per-GPU attention work of the configs
ATTN = [
    ("c1 tiny 256x6h d64", [256], 6, 64),
    ("c2 4x4096 12h", [4096] * 4, 12, 128),
    ("c3 480p sp1 12h", [32760], 12, 128),
    ("c3 480p sp8 2h", [32760], 2, 128),
    ("c4 720p sp8 5h", [75600], 5, 128),
    ("c4 720p sp2 20h", [75600], 20, 128),
    ("c4 720p sp1 40h", [75600], 40, 128),
]
# (label, M, N, K)
GEMM = [
    ("c2 qkv", 16384, 4608, 1536), ("c2 o", 16384, 1536, 1536), ("c2 up", 16384, 8960, 1536),
    ("c2 down", 16384, 1536, 8960),
    ("c4 sp8 qkv", 9450, 15360, 5120), ("c4 sp8 o", 9450, 5120, 5120),
    ("c4 sp8 up", 9450, 13824, 5120), ("c4 sp8 down", 9450, 5120, 13824),
    ("c4 sp1 qkv", 75600, 15360, 5120), ("c4 cfg qkv", 151200, 15360, 5120), ("c4 sp1 up", 75600, 13824, 5120),
    ("c4 cfg up", 151200, 13824, 5120),
    ("c3 sp8 qkv", 4095, 4608, 1536), ("c3 sp8 o", 4095, 1536, 1536), ("c3 sp8 up", 4095, 8960, 1536),
    ("c3 sp8 down", 4095, 1536, 8960), ("c3 sp4 o", 8190, 1536, 1536), ("c3 sp4 down", 8190, 1536, 8960),
]


def timeit(ctx, fn, reps):
    s = torch.cuda.ExternalStream(ctx.stream_ptr(0))
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--attn", action="store_true")
    ap.add_argument("--gemm", action="store_true")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--torch", action="store_true", help="also time torch SDPA / matmul yardsticks")
    ap.add_argument("--only", default=None, help="substring filter on the case label")
    ap.add_argument("--lib", default=None, help="load this libgs.so instead of the in-tree one (A/B)")
    ap.add_argument("--epi", default="bf16", choices=["bf16", "gelu", "resid"],
                    help="GEMM epilogue: bf16 out, GELU bf16 out, or fp32 gated residual x += g (acc + b)")
    a = ap.parse_args()
    if a.lib:
        gs.load(a.lib)
    if not (a.attn or a.gemm):
        a.attn = a.gemm = True
    ctx = gs.Context(device=0)
    res = {}
    if a.attn:
        for label, seqs, H, d in ATTN:
            if a.only and a.only not in label:
                continue
            N = sum(seqs)
            q = torch.randn(N, H, d, device="cuda").to(torch.bfloat16)
            k = torch.randn(N, H, d, device="cuda").to(torch.bfloat16)
            v = torch.randn(N, H, d, device="cuda").to(torch.bfloat16)
            o = torch.empty_like(q)
            offs = list(np.cumsum([0] + seqs[:-1]))
            ms = timeit(ctx, lambda: ctx.debug_attention(q, k, v, o, H, d, offs, seqs), a.reps)
            fl = 4 * d * H * sum(n * n for n in seqs)
            tf = fl / ms / 1e9
            line = f"attn {label:24s} {ms:9.3f} ms {tf:8.1f} TFLOP/s {tf / PEAK:6.1%} of peak"
            if a.torch:
                qq = q.permute(1, 0, 2)[None]
                kk = k.permute(1, 0, 2)[None]
                vv = v.permute(1, 0, 2)[None]
                if len(seqs) == 1:
                    f = lambda: torch.nn.functional.scaled_dot_product_attention(qq, kk, vv)
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    f()
                    e0.record()
                    for _ in range(a.reps):
                        f()
                    e1.record()
                    torch.cuda.synchronize()
                    tms = e0.elapsed_time(e1) / a.reps
                    line += f" | torch sdpa {tms:8.3f} ms {fl / tms / 1e9:7.1f}"
            print(line, flush=True)
            res[label] = tf
            del q, k, v, o
    if a.gemm:
        for label, M, N, K in GEMM:
            if a.only and a.only not in label:
                continue
            A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
            W = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
            b = torch.zeros(N, device="cuda").to(torch.bfloat16)
            if a.epi == "resid":
                out = torch.zeros(M, N, device="cuda", dtype=torch.float32)
                ga = torch.rand(N, device="cuda")
                gb = torch.rand(4, N, device="cuda")
                rr = (torch.arange(M, device="cuda", dtype=torch.int32) * 4) // M
                fn = lambda: ctx.debug_gemm(gs.EPI_RESID_F32, M, N, K, A, W, b, out, ga, gb, N, rr)
            else:
                out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
                e = gs.EPI_GELU_BF16 if a.epi == "gelu" else gs.EPI_BF16
                fn = lambda: ctx.debug_gemm(e, M, N, K, A, W, b, out)
            ms = timeit(ctx, fn, a.reps)
            tf = 2 * M * N * K / ms / 1e9
            line = f"gemm {label:24s} {ms:9.3f} ms {tf:8.1f} TFLOP/s {tf / PEAK:6.1%} of peak"
            if a.torch:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.matmul(A, W.t())
                e0.record()
                torch.matmul(A, W.t())
                e1.record()
                torch.cuda.synchronize()
                tms = e0.elapsed_time(e1)
                line += f" | cublas {tms:8.3f} ms {2 * M * N * K / tms / 1e9:7.1f}"
            print(line, flush=True)
            res[label] = tf
            del A, W, out
    ctx.close()


if __name__ == "__main__":
    main()
