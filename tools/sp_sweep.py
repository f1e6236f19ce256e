"""Per-GPU work of a DiT step at SP degree p = 1, 2, 4, 8, emulated on one B200 (p virtual ranks
run one after another on the same device, fused peer-store exchange in emulated mode).  For each
(config, p) it reports the device time of the whole step summed over the p positions, divided by
p (= one GPU's compute share when the work is balanced), and the all-to-all bytes one GPU sends per
step (4 (p-1)/p (n/p) D 2 per block) with the time they would take at 900 GB/s
per direction of NVLink 5.  A projection for the multi-GPU step, not a multi-GPU measurement.
  python tools/sp_sweep.py [--layers 4] [--configs c3,c4]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2604_04335_b200 as gs  # noqa: E402
from synth import models as sm  # noqa: E402

CONFIGS = {"c3": (sm.WAN_1_3B, 832, 480, 81), "c4": (sm.WAN_14B, 1280, 720, 81)}
NVLINK_GBS = 900.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--configs", default="c3,c4")
    a = ap.parse_args()
    out = {"how": __doc__.split("\n\n")[0].replace("\n", " "), "layers": a.layers, "rows": []}
    for cname in a.configs.split(","):
        base, w, h, f = CONFIGS[cname]
        shape = base.with_layers(a.layers)
        n = int(np.prod(sm.token_grid(w, h, f)))
        for p in (1, 2, 4, 8):
            ctx = gs.Context(device=0, world_size=8, emulated=True)
            ctx.set_option("a2a", 1)
            mid = ctx.model_create(shape.dim, shape.heads, shape.ffn, shape.layers, shape.weight_seed)
            ranks = list(range(p))
            req = ctx.submit(mid, w, h, f, 50, 1000, ranks)
            ctx.run_steps([req], ranks, 1)  # warm-up
            ctx.profile(1, True)
            ctx.run_steps([req], ranks, 2)
            st = ctx.stats()
            ctx.close()
            per = {k: st[k]["ms"] / 2 for k in st if isinstance(st[k], dict) and not k.startswith("_")}
            total = sum(per.values())
            a2a_bytes = 4 * (p - 1) / p * (n / p) * shape.dim * 2 * a.layers
            row = {"config": cname, "p": p, "tokens": n, "per_gpu_ms_per_step": round(total / p, 2),
                   "attention_ms_per_gpu": round(per.get("attention", 0.0) / p, 2),
                   "gemm_ms_per_gpu": round(sum(v for k, v in per.items() if k.startswith("gemm")) / p, 2),
                   "a2a_bytes_per_gpu": int(a2a_bytes),
                   "a2a_ms_at_nvlink": round(a2a_bytes / (NVLINK_GBS * 1e9) * 1e3, 2),
                   "speedup_vs_p1_compute": None}
            out["rows"].append(row)
            print(json.dumps(row), flush=True)
        rows = [r for r in out["rows"] if r["config"] == cname]
        for r in rows:
            r["speedup_vs_p1_compute"] = round(rows[0]["per_gpu_ms_per_step"] / r["per_gpu_ms_per_step"], 3)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
