"""Per-tile timeline of the first attention CTA (GS_ATTN_TRACE=1): MMA issue, softmax wake/load/done."""
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
QKV = (q, k, v)
for _ in range(2):
    ctx.debug_attention(q, k, v, o, H, d, [0], [N])
t = ctx.debug_attention_trace().astype(np.int64)
t0 = t[t > 0].min()
names = ["issue_S", "issue_PV", "sm_wake", "sm_loaded", "Pdone_q0", "Pdone_q1", "Pdone_q2", "Pdone_q3"]
print("tile  " + "  ".join(f"{n}{w:>1d}".rjust(11) for n in names for w in range(2)))
for j in range(32):
    print(f"{j:4d}  " + "  ".join(f"{(t[e, j, w] - t0) if t[e, j, w] else -1:11d}" for e in range(8) for w in range(2)))
d_ = np.diff(t[2, 4:30, 0])
print("WG0 period (cycles) median", np.median(d_))
print("softmax T_s (wake->Pdone) median", np.median(t[4, 4:30, 0] - t[2, 4:30, 0]),
      "load", np.median(t[3, 4:30, 0] - t[2, 4:30, 0]))
print("Pdone -> issue_PV median", np.median(t[1, 4:30, 0] - t[4, 4:30, 0]))
for q in range(4):
    print(f"WG0 q{q} T_s median", np.median(t[4 + q, 4:30, 0] - t[2, 4:30, 0]),
          f"WG1 q{q} T_s median", np.median(t[4 + q, 4:30, 1] - t[2, 4:30, 1]))
print("issue_S(j+1) -> wake(j+1) median", np.median(t[2, 5:30, 0] - t[0, 5:30, 0]))
print("issue_S: kfull wait (cycles) median", np.median(t[0, 4:30, 0] - t[11, 4:30, 0]), np.median(t[0, 4:30, 1] - t[11, 4:30, 1]))
print("issue_PV: vfull+pfull wait median", np.median(t[10, 4:30, 0] - t[12, 4:30, 0]), np.median(t[10, 4:30, 1] - t[12, 4:30, 1]))
print("PV0 issue -> S0(j+1) pre-wait median", np.median(t[11, 5:30, 0] - t[1, 4:29, 0]))
print("timeline (cycles rel. to issue_PV0(j) start), WG0 then WG1:")
for j in range(20, 24):
    for w in range(2):
        b = t[1, j, w]
        ev = [("PV_issue_end", t[14, j, w]), ("S(j+1)_issue", t[0, j + 1, w]), ("S(j+1)_issue_end", t[13, j + 1, w]),
              ("wake(j+1)", t[2, j + 1, w]), ("loaded", t[3, j + 1, w]),
              ("Pdone q0..q3", max(t[4 + q, j + 1, w] for q in range(4))), ("pfull_ok", t[10, j + 1, w]),
              ("PV(j+1)_issue", t[1, j + 1, w])]
        print(f" j={j} WG{w}: " + ", ".join(f"{n} {v - b:+d}" for n, v in ev))
for j in range(20, 24):
    b = t[1, j, 0]
    print(f" loop head j={j}: start {t[15, j, 0] - b:+d} kv-ok {t[11, j, 0] - b:+d} "
          f"pfull0-ok {t[10, j, 0] - b:+d}  (prev S0 issue end {t[13, j, 0] - b:+d})")
for j in range(20, 26):
    print(f"tile {j}: K issued {t[8, j, 0] - t0}  V issued {t[9, j, 0] - t0}  MMA pfull0-ok {t[10, j, 0] - t0} "
          f"PV0 issued {t[1, j, 0] - t0}  pfull1-ok {t[10, j, 1] - t0} PV1 issued {t[1, j, 1] - t0}")
ctx.close()

# pair peer (CTA 1): its clock64 is another SM's counter, so compare durations, not stamps
if d == 128:
    ctx2 = gs.Context(device=0)
    for _ in range(2):
        ctx2.debug_attention(*QKV, o, H, d, [0], [N])
    t0s = ctx2.debug_attention_trace(0).astype(np.int64)
    t1s = ctx2.debug_attention_trace(1).astype(np.int64)
    for name, tt in (("leader", t0s), ("peer", t1s)):
        print(f"{name}: period {np.median(np.diff(tt[2, 4:30, 0]))} T_s {np.median(tt[4:8, 4:30, 0].max(0) - tt[2, 4:30, 0])}"
              f" T_s WG1 {np.median(tt[4:8, 4:30, 1].max(0) - tt[2, 4:30, 1])}")
    # offset estimate: wake events of both CTAs are triggered by the same multicast commit
    off = np.median(t1s[2, 4:30, 0] - t0s[2, 4:30, 0])
    print("peer clock offset (from wake of WG0, assumes simultaneous wake)", off)
    for j in range(20, 24):
        for w in range(2):
            print(f" j={j} WG{w}: leader wake {t0s[2, j, w] - t0s[1, j, 0]:+d} Pdone {t0s[4:8, j, w].max() - t0s[1, j, 0]:+d}"
                  f" | peer wake {t1s[2, j, w] - off - t0s[1, j, 0]:+.0f} Pdone {t1s[4:8, j, w].max() - off - t0s[1, j, 0]:+.0f}"
                  f" | leader pfull_ok {t0s[10, j, w] - t0s[1, j, 0]:+d}")
    ctx2.close()

print("MMA-thread timeline rel. to PV0(j) issue: head, kv-ok | wait_p0, p0-ok, PV0 issue..end, S0(j+1) issue..end |"
      " wait_p1, p1-ok, PV1 issue..end, S1(j+1) issue..end")
for j in range(20, 24):
    b = t[1, j, 0]
    r = lambda e, w, jj=j: t[e, jj, w] - b  # noqa: E731
    print(f" j={j}: {r(15, 0):+d} {r(11, 0):+d} | {r(12, 0):+d} {r(10, 0):+d} {r(1, 0):+d}..{r(14, 0):+d} "
          f"{r(0, 0, j + 1):+d}..{r(13, 0, j + 1):+d} | {r(12, 1):+d} {r(10, 1):+d} {r(1, 1):+d}..{r(14, 1):+d} "
          f"{r(0, 1, j + 1):+d}..{r(13, 1, j + 1):+d} | Pdone WG0 {t[4:8, j, 0].max() - b:+d} WG1 {t[4:8, j, 1].max() - b:+d}")
