"""Per-tile timeline of the first CTA pair of the alternating-set attention variant (libgs_alt.so,
built with -DGS_ATTN_ALT=1; GS_ATTN_TRACE=1): issuer S / PV issue, softmax wake / loaded / max /
exchange / exp done / P arrive per KV tile (tile j -> softmax set j & 1, S/P buffer j % 3)."""
import os
import sys

os.environ["GS_ATTN_TRACE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("GS_LIB", os.path.join(ROOT, "paper_2604_04335_b200", "libgs_alt.so"))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2604_04335_b200 as gs  # noqa: E402

ctx = gs.Context(device=0)
N, H, d = 75600, 5, 128
q, k, v = (torch.randn(N, H, d, device="cuda").to(torch.bfloat16) for _ in range(3))
o = torch.empty_like(q)
for _ in range(2):
    ctx.debug_attention(q, k, v, o, H, d, [0], [N])
ev = {"issS": 0, "Vok": 7, "issPV": 1, "wake": 2, "loaded": 3, "max": 4, "xchg": 5, "exp": 6,
      "arr_q0": 8, "arr_q1": 9, "arr_q2": 10, "arr_q3": 11}
for cta in range(2):
    t = ctx.debug_attention_trace(cta).astype(np.int64)[:, :, 0]  # [event][tile]
    ok = t[t > 0]
    if ok.size == 0:
        continue
    t0 = ok.min()
    print(f"CTA {cta}")
    print("tile " + "".join(f"{n:>9s}" for n in ev))
    for j in range(0, 24):
        print(f"{j:4d} " + "".join(f"{(t[e, j] - t0) if t[e, j] else -1:9d}" for e in ev.values()))
    sl = slice(6, 30)
    print("tile period wake(j)->wake(j+1) median", np.median(np.diff(t[2, 6:30])))
    print("same-set period wake(j)->wake(j+2) median", np.median(t[2, 8:30] - t[2, 6:28]))
    for a, b in (("wake", "loaded"), ("loaded", "max"), ("max", "xchg"), ("xchg", "exp"), ("exp", "arr_q0")):
        print(f"  {a:>6s} -> {b:<6s} median {np.median(t[ev[b], sl] - t[ev[a], sl]):8.1f}")
    if cta == 0:
        arr = t[8:12, sl].max(0)
        print("  last arrive -> issPV", np.median(t[1, sl] - arr))
        print("  issPV(j) -> issS(j+3)", np.median(t[0, 9:30] - t[1, 6:27]))
        print("  issS(j) -> wake(j)", np.median(t[2, sl] - t[0, sl]))
        print("  P_j arrive -> wake(j+2) (set idle)", np.median(t[2, 8:30] - t[8:12, 6:28].max(0)))
ctx.close()
