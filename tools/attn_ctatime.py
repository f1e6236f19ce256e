"""Per-CTA timing of one attention launch (GS_ATTN_TRACE=1): CTA duration, prologue (entry ->
first S issued), and the gap between consecutive CTAs on an SM -- the fixed per-CTA cost that
short sequences (config 2: 4 x 4096 tokens) pay.
  python tools/attn_ctatime.py [--seq 4096 --nreq 4 --heads 12]"""
import argparse
import os
import sys

os.environ["GS_ATTN_TRACE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2604_04335_b200 as gs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seq", type=int, default=4096)
ap.add_argument("--nreq", type=int, default=4)
ap.add_argument("--heads", type=int, default=12)
a = ap.parse_args()
ctx = gs.Context(device=0)
N, H, d = a.seq * a.nreq, a.heads, 128
q, k, v = (torch.randn(N, H, d, device="cuda").to(torch.bfloat16) for _ in range(3))
o = torch.empty_like(q)
offs = [i * a.seq for i in range(a.nreq)]
for _ in range(3):
    ctx.debug_attention(q, k, v, o, H, d, offs, [a.seq] * a.nreq)
ncta = 2 * ((a.seq + 511) // 512) * a.nreq * H
t = ctx.debug_attention_ctatime(min(ncta, 8192)).astype(np.int64)
t0 = t[:, 0].min()
dur = (t[:, 2] - t[:, 0]) / 1e3
pro = (t[0::2, 1] - t[0::2, 0]) / 1e3
print(f"{len(t)} CTAs, launch span {(t[:, 2].max() - t0) / 1e3:.1f} us")
print(f"CTA duration us: median {np.median(dur):.1f} min {dur.min():.1f} max {dur.max():.1f}")
print(f"prologue (entry -> first S issued) us: median {np.median(pro):.2f} max {pro.max():.2f}")
gaps, busy = [], []
for sm in np.unique(t[:, 3]):
    r = t[t[:, 3] == sm]
    r = r[np.argsort(r[:, 0])]
    busy.append((r[:, 2] - r[:, 0]).sum())
    gaps += list((r[1:, 0] - r[:-1, 2]) / 1e3)
span = t[:, 2].max() - t0
print(f"inter-CTA gap on an SM us: median {np.median(gaps):.2f} max {np.max(gaps):.2f}")
print(f"SM busy fraction of the span: mean {np.mean(busy) / span:.3f}")
ctx.close()
