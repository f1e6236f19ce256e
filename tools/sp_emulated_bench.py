"""Single-GPU look at the SP exchange cost: one 720p Wan-14B step (config 4) at SP = p emulated on
one B200 (p virtual ranks, executed one after another), transfer plans (a2a = 0: pack into send
buffers + device copies + O staging / unpack) vs fused peer stores (a2a = 1: the pack kernel and
the attention epilogue write the consumers' buffers directly).  Prints per-class device time
(gs_stats, CUDA events on the context stream) summed over the p positions; the step time is
p x the per-GPU work, not a multi-GPU number.
  python tools/sp_emulated_bench.py [--p 8] [--layers 4]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_04335_b200 as gs  # noqa: E402
from synth import models as sm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--p", type=int, default=8)
    ap.add_argument("--layers", type=int, default=4)
    a = ap.parse_args()
    shape = sm.WAN_14B.with_layers(a.layers)
    out = {}
    for mode in (0, 1):
        ctx = gs.Context(device=0, world_size=8, emulated=True)
        ctx.set_option("a2a", mode)
        mid = ctx.model_create(shape.dim, shape.heads, shape.ffn, shape.layers, shape.weight_seed)
        ranks = list(range(a.p))
        req = ctx.submit(mid, 1280, 720, 81, 50, 1000, ranks)
        ctx.run_steps([req], ranks, 1)  # warm-up (allocations, IPC-free in emulated mode)
        ctx.profile(True, True)
        ctx.run_steps([req], ranks, 2)
        st = ctx.stats()
        ctx.close()
        keys = [k for k in st if isinstance(st[k], dict)]
        per = {k: round(st[k]["ms"] / 2, 3) for k in sorted(keys)}
        exch = sum(v for k, v in per.items() if k.startswith("a2a"))
        out["peer" if mode else "plans"] = {"ms_per_step_by_class": per, "exchange_ms": round(exch, 3),
                                            "qk_norm_rope_pack_ms": per.get("qk_norm_rope"),
                                            "attention_ms": per.get("attention")}
    print(json.dumps({"workload": f"t2v720 Wan-14B {a.layers} layers, SP={a.p} emulated on 1 GPU", **out},
                     indent=1))


if __name__ == "__main__":
    main()
