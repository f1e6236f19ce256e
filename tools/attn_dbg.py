import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2604_04335_b200 as gs
from oracle import dit
from tests.gpu_util import from_dev_bf16, rel_l2
ctx = gs.Context(device=0)
for (seqlens, H) in [([75600], 5), ([32760], 12), ([4096, 3840, 3840, 4032], 12), ([75600], 40), ([2000], 5), ([2000], 12), ([20000], 12)]:
    d = 128
    g = torch.Generator(device="cuda").manual_seed(1)
    N = sum(seqlens)
    q, k, v = (torch.randn(N, H, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    off = np.cumsum([0] + seqlens[:-1]).tolist()
    outs = []
    for rep in range(3):
        o = torch.zeros_like(q)
        ctx.debug_attention(q, k, v, o, H, d, off, seqlens)
        outs.append(o.clone())
    same = all(torch.equal(outs[0].view(torch.int16), x.view(torch.int16)) for x in outs[1:])
    qf, kf, vf = (from_dev_bf16(t) for t in (q, k, v))
    got = from_dev_bf16(outs[0])
    errs = []
    for o_, n in zip(off, seqlens):
        rows = np.array([0, 1, 100, 127, 128, 200, 255, 256, 300, n // 2, n - 1])
        ref = dit.attention(qf[o_ + rows], kf[o_:o_ + n], vf[o_:o_ + n])
        per = [rel_l2(got[o_ + r], ref[i]) for i, r in enumerate(rows)]
        errs.append(np.round(per, 3).tolist())
    print(seqlens[:2], H, 'deterministic' if same else 'NONDETERMINISTIC', errs, flush=True)
