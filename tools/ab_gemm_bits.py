"""A/B bit check of the GEMM epilogues between two builds of libgs.so (development aid).

  python tools/ab_gemm_bits.py --lib A.so --out a.npz ; python tools/ab_gemm_bits.py --lib B.so --out b.npz
  python tools/ab_gemm_bits.py --compare a.npz b.npz

Runs every epilogue kind on seeded inputs at ragged shapes (M not a multiple of the 256-row pair
tile, several N tiles, 192- and 256-wide tiles) and stores the outputs' SHA-256 digests.
"""
import argparse
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

SHAPES = [(300, 256, 128), (1000, 1536, 1536), (4095, 1536, 1536), (777, 4608, 256), (513, 64, 1536)]


def run(lib, out):
    import torch
    import paper_2604_04335_b200 as gs
    if lib:
        gs.load(lib)
    ctx = gs.Context(device=0)
    res = {}
    for (M, N, K) in SHAPES:
        g = torch.Generator(device="cuda").manual_seed(M * 7 + N * 3 + K)
        A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
        W = (torch.randn(N, K, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
        b = (torch.randn(N, device="cuda", generator=g) * 0.1).to(torch.bfloat16)
        ga = torch.rand(N, device="cuda", generator=g)
        gb = torch.rand(3, N, device="cuda", generator=g)
        rr = ((torch.arange(M, device="cuda") * 3) // M).to(torch.int32)
        x0 = torch.randn(M, N, device="cuda", generator=g)
        for bn in (0, 192, 256):
            if bn == 192 and N % 192:
                continue
            ctx.set_option("gemm_bn", bn)
            for e in range(6):
                if e in (0, 1):
                    o = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
                    ctx.debug_gemm(e, M, N, K, A, W, b, o)
                elif e == 2:
                    o = torch.empty(M, N, device="cuda")
                    ctx.debug_gemm(e, M, N, K, A, W, b, o)
                else:
                    o = x0.clone()
                    ctx.debug_gemm(e, M, N, K, A, W, b, o, ga, gb, N, rr, dsig=[0.1, -0.2, 0.3])
                torch.cuda.synchronize()
                res[f"{M}x{N}x{K} bn{bn} epi{e}"] = hashlib.sha256((o.view(torch.int16) if o.dtype == torch.bfloat16 else o).cpu().numpy().tobytes()).hexdigest()
    ctx.set_option("gemm_bn", 0)
    ctx.close()
    np.savez(out, **{k: np.array(v) for k, v in res.items()})
    print(f"{len(res)} digests -> {out}")


def compare(a, b):
    A, B = np.load(a), np.load(b)
    bad = [k for k in A.files if str(A[k]) != str(B[k])]
    print(f"{len(A.files)} cases, {len(bad)} differ" + ("".join("\n  " + k for k in bad)))
    return 1 if bad else 0


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=None)
    ap.add_argument("--out", default="gpurun_out/gemm_bits.npz")
    ap.add_argument("--compare", nargs=2, default=None)
    a = ap.parse_args()
    sys.exit(compare(*a.compare) if a.compare else run(a.lib, a.out))
