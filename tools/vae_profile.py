"""VAE decode profile (development aid): wall time of the Wan-VAE-shaped 720p/81f decode and of each
convolution shape class, by timing gs_debug_conv3d at the decoder's layer shapes.
  python tools/vae_profile.py [--once]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2604_04335_b200 as gs  # noqa: E402
from paper_2604_04335_b200 import costmodel  # noqa: E402

once = "--once" in sys.argv
ctx = gs.Context(device=0)
vid = ctx.vae_create()
grid = (21, 45, 80)
lat = torch.randn(int(np.prod(grid)) * 64, device="cuda")
out = torch.empty(ctx.vae_out_shape(grid), device="cuda")
ctx.vae_decode(vid, lat, grid, out=out)
if once:
    sys.exit(0)
torch.cuda.synchronize()
t0 = time.perf_counter()
ctx.vae_decode(vid, lat, grid, out=out)
torch.cuda.synchronize()
ms = (time.perf_counter() - t0) * 1e3
fl = costmodel.vae_decode_flops(grid)
print(f"decode 720p/81f: {ms:.1f} ms, {fl / ms / 1e9:.1f} TFLOP/s algorithmic")
ctx.close()
# per-shape conv timing (T, H, W, Cp, k, Coutp): the decoder's dominant layer shapes
ctx = gs.Context(device=0)
shapes = [("stage3 3x3x3 96->96", 81, 720, 1280, 96, (3, 3, 3), 96),
          ("stage2 3x3x3 192->192", 81, 360, 640, 192, (3, 3, 3), 192),
          ("stage2 sconv 1x3x3 192->96", 81, 720, 1280, 192, (1, 3, 3), 96),
          ("stage1 3x3x3 384->384", 41, 180, 320, 384, (3, 3, 3), 384),
          ("stage0 3x3x3 384->384", 21, 90, 160, 384, (3, 3, 3), 384)]
for name, T, H, W, C, k, Co in shapes:
    if T * H * W * max(C, Co) * 2 > 40e9:
        continue
    x = torch.randn(T, H, W, C, device="cuda").to(torch.bfloat16)
    w = (torch.randn(Co, *k, C, device="cuda") * 0.02).to(torch.bfloat16)
    b = torch.zeros(Co, device="cuda").to(torch.bfloat16)
    o = torch.empty(T, H, W, Co, device="cuda", dtype=torch.bfloat16)
    ctx.debug_conv3d(x, w, b, o, T, H, W, C, k, Co)
    torch.cuda.synchronize()
    a = time.perf_counter()
    ctx.debug_conv3d(x, w, b, o, T, H, W, C, k, Co)
    torch.cuda.synchronize()
    cms = (time.perf_counter() - a) * 1e3
    f = 2 * T * H * W * C * Co * k[0] * k[1] * k[2]
    print(f"conv {name:36s} {cms:8.2f} ms {f / cms / 1e9:8.1f} TFLOP/s")
    del x, w, b, o
    torch.cuda.empty_cache()
ctx.close()
