"""Start-up ramp of the ping-pong in the first attention CTA (GS_ATTN_TRACE=1): per KV tile the
two softmax groups' wake times, their offset, and the per-group period (config-2 shape by
default: a request's 32 KV tiles)."""
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
ap.add_argument("--heads", type=int, default=12)
a = ap.parse_args()
ctx = gs.Context(device=0)
N, H, d = a.seq, a.heads, 128
q, k, v = (torch.randn(N, H, d, device="cuda").to(torch.bfloat16) for _ in range(3))
o = torch.empty_like(q)
for _ in range(3):
    ctx.debug_attention(q, k, v, o, H, d, [0], [N])
t = ctx.debug_attention_trace(0).astype(np.int64)  # [event][tile][group]
t0 = t[t > 0].min()
nt = min(32, (N + 127) // 128)
print("tile  wake0   wake1   off(w1-w0)  Pdone0  Pdone1  period0 period1")
for j in range(nt):
    w0, w1 = t[2, j, 0] - t0, t[2, j, 1] - t0
    p0, p1 = t[4:8, j, 0].max() - t0, t[4:8, j, 1].max() - t0
    per0 = (t[2, j + 1, 0] - t[2, j, 0]) if j + 1 < nt else 0
    per1 = (t[2, j + 1, 1] - t[2, j, 1]) if j + 1 < nt else 0
    print(f"{j:4d} {w0:7d} {w1:7d} {w1 - w0:8d} {p0:8d} {p1:8d} {per0:7d} {per1:7d}")
ctx.close()
