"""Yardstick profile (development aid): torch SDPA (cuDNN backend) at the c4 SP=8 attention shape,
for ncu: 75600 tokens, 5 heads, d = 128, bf16."""
import torch
from torch.nn.attention import SDPBackend, sdpa_kernel

N, H, d = 75600, 5, 128
q, k, v = (torch.randn(1, H, N, d, device="cuda", dtype=torch.bfloat16) for _ in range(3))
with sdpa_kernel(SDPBackend.CUDNN_ATTENTION):
    for _ in range(3):
        o = torch.nn.functional.scaled_dot_product_attention(q, k, v)
torch.cuda.synchronize()
print("ok", o.shape)
