"""One stage-3-shaped VAE conv (81 x 720 x 1280, 96 -> 96, 3x3x3) for ncu (development aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_04335_b200 as gs  # noqa: E402

T, H, W, C, Co = (int(a) for a in (sys.argv[1:6] if len(sys.argv) > 5 else (21, 720, 1280, 96, 96)))
ctx = gs.Context(device=0)
x = torch.randn(T, H, W, C, device="cuda").to(torch.bfloat16)
w = (torch.randn(Co, 3, 3, 3, C, device="cuda") * 0.02).to(torch.bfloat16)
b = torch.zeros(Co, device="cuda").to(torch.bfloat16)
o = torch.empty(T, H, W, Co, device="cuda", dtype=torch.bfloat16)
for _ in range(2):
    ctx.debug_conv3d(x, w, b, o, T, H, W, C, (3, 3, 3), Co)
torch.cuda.synchronize()
ctx.close()
print("ok")
