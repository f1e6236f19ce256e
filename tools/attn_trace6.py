"""Per-tile timeline of the first v6 attention CTA (GS_ATTN_TRACE=1, single softmax group, S/P
double-buffered): MMA issue S / PV, issuer sees P, softmax wake / loaded / P done."""
import os
import sys

os.environ["GS_ATTN_TRACE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
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
for cta in range(2):
    t = ctx.debug_attention_trace(cta).astype(np.int64)[:, :, 0]  # [event][tile]
    ok = t[t > 0]
    if ok.size == 0:
        continue
    t0 = ok.min()
    ev = {"issue_S": 0, "issue_PV": 1, "P_seen": 10, "wake": 2, "loaded": 3, "Pd_q0": 4, "Pd_q1": 5,
          "Pd_q2": 6, "Pd_q3": 7}
    print(f"CTA {cta}")
    print("tile " + "".join(f"{n:>10s}" for n in ev))
    for j in range(4, 14):
        print(f"{j:4d} " + "".join(f"{(t[e, j] - t0) if t[e, j] else -1:10d}" for e in ev.values()))
    sl = slice(6, 30)
    print("period (wake j -> wake j+1) median", np.median(np.diff(t[2, 6:30])))
    print("softmax wake->Pdone(max q) median", np.median(t[4:8, sl].max(0) - t[2, sl]),
          "wake->loaded", np.median(t[3, sl] - t[2, sl]))
    print("Pdone(max q) -> P_seen", np.median(t[10, sl] - t[4:8, sl].max(0)),
          "P_seen -> issue_PV", np.median(t[1, sl] - t[10, sl]))
    print("issue_S(j+2) -> wake(j+2)", np.median(t[2, 8:30] - t[0, 8:30]),
          "Pdone(j) -> wake(j+1)", np.median(t[2, 7:31] - t[4:8, 6:30].max(0)))
    if cta == 0:
        print("issue_PV(j) -> issue_PV(j+1)", np.median(np.diff(t[1, 6:30])))
    ph = [("loaded", 3), ("max", 11), ("xchg", 12), ("pbuf", 13), ("exp", 14), ("Pdone", 4)]
    prev = t[2, sl]
    for n, e in ph:
        print(f"  warp0 phase -> {n:6s} median {np.median(t[e, sl] - prev):7.1f}")
        prev = t[e, sl]
ctx.close()
