"""A/B bit check of whole DiT steps between two libgs.so builds (GS_LIB selects the build):
`python tools/ab_step_bits.py dump out.npz` under each build, then `compare a.npz b.npz`.
Cases: ragged varlen batches of the tiny / Wan-1.3B / Wan-14B shapes at SP 1, 2 (peer-store
pack) and 8 (uneven heads), 2 steps each after a 1-step offset of the first request."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CASES = [  # (model, layers, requests (w, h, frames), SP degree, a2a mode: 1 peer stores, 0 transfer plans)
    ("tiny", 2, [(256, 256, 1), (320, 192, 1), (160, 96, 1)], 1, 1),
    ("wan-1.3b", 2, [(256, 256, 1), (320, 192, 1), (416, 240, 5)], 1, 1),
    ("wan-1.3b", 1, [(416, 240, 5), (256, 256, 1)], 2, 1),
    ("wan-1.3b", 1, [(416, 240, 5), (256, 256, 1)], 4, 0),
    ("wan-1.3b", 1, [(416, 240, 5)], 8, 1),
    ("wan-14b", 1, [(320, 176, 5), (256, 256, 1)], 2, 1),
    ("wan-14b", 1, [(320, 176, 5), (16, 16, 1)], 8, 0),
]


def dump(path):
    import paper_2604_04335_b200 as gs
    from synth import models as sm
    out = {}
    for ci, (name, layers, sizes, p, a2a) in enumerate(CASES):
        shape = sm.MODELS[name].with_layers(layers)
        ctx = gs.Context(device=0, world_size=8, emulated=True)
        ctx.set_option("a2a", a2a)
        mid = ctx.model_create(shape.dim, shape.heads, shape.ffn, shape.layers, shape.weight_seed)
        ranks = list(range(p))
        reqs = [ctx.submit(mid, w, h, f, 50, 1000 + i, ranks) for i, (w, h, f) in enumerate(sizes)]
        ctx.run_steps([reqs[0]], ranks, 1)
        ctx.run_steps(reqs, ranks, 2)
        for ri, r in enumerate(reqs):
            out[f"c{ci}_r{ri}"] = ctx.read_latent(r)
        ctx.close()
    np.savez(path, **out)
    print(f"dumped {len(out)} latents to {path} (lib {os.environ.get('GS_LIB', 'in-tree')})")


def compare(a, b):
    A, B = np.load(a), np.load(b)
    bad = [k for k in A.files if not np.array_equal(A[k].view(np.uint32), B[k].view(np.uint32))]
    print(f"{len(A.files) - len(bad)}/{len(A.files)} latents bit-identical" + (f"; differ: {bad}" if bad else ""))
    return 1 if bad else 0


if __name__ == "__main__":
    if sys.argv[1] == "dump":
        dump(sys.argv[2])
    else:
        sys.exit(compare(sys.argv[2], sys.argv[3]))
