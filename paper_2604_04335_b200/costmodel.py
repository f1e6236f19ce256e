"""Algorithmic work accounting for the DiT-step hot path (bench.py denominators).

Not the method's arithmetic: this counts FLOPs and bytes.  The paper's own per-step cost
model (Tab. `arithmetic_intensity`) is reproduced exactly by

    FLOPs/step = L * (8 N D^2 + 4 N^2 D + 4 N D F)
    bytes/step = L * (2 (4 D^2 + 2 D F) + 12 N D)

(SURVEY.md §0 / §8(c) pin P1; tests/test_costmodel.py checks all 12 printed values).
Varlen batches replace N^2 by sum_r n_r^2 in the attention term (block-diagonal).
"""


def gemm_flops_per_block(n_tokens, dim, ffn):
    """QKV + O + MLP up/down: 2*N*(3D*D + D*D + 2*D*F) = 8 N D^2 + 4 N D F."""
    return 8 * n_tokens * dim * dim + 4 * n_tokens * dim * ffn


def attn_flops_per_block(seqlens, dim):
    """QK^T + PV over all heads: 4 * D * sum_r n_r^2 (softmax work not counted)."""
    return 4 * dim * sum(n * n for n in seqlens)


def flops_per_block(seqlens, dim, ffn):
    return gemm_flops_per_block(sum(seqlens), dim, ffn) + attn_flops_per_block(seqlens, dim)


def paper_flops_per_step(layers, n_tokens, dim, ffn):
    """Tab. arithmetic_intensity FLOPs/step (one forward, self-attn + MLP)."""
    return layers * (8 * n_tokens * dim ** 2 + 4 * n_tokens ** 2 * dim + 4 * n_tokens * dim * ffn)


def paper_bytes_per_step(layers, n_tokens, dim, ffn):
    """Tab. arithmetic_intensity bytes/step: bf16 weights + 12 N D activation bytes per block."""
    return layers * (2 * (4 * dim ** 2 + 2 * dim * ffn) + 12 * n_tokens * dim)


def elementwise_bytes_per_token(dim):
    """HBM bytes per token per block of the element-wise kernels:
    LN1+mod reads x fp32 (4D) writes a bf16 (2D); qk-RMSNorm+RoPE reads q,k bf16 (4D)
    writes them (4D); LN2+mod as LN1 (6D)."""
    return 6 * dim + 8 * dim + 6 * dim


def a2a_bytes_per_rank(n_tokens, dim, p):
    """Ulysses all-to-all bytes sent per rank per block: (Q,K,V fwd + O back) * (p-1)/p."""
    local = n_tokens / p
    return 4 * (p - 1) / p * local * dim * 2


def vae_decode_flops(grid, dims=(384, 384, 384, 192, 96), blocks=3, mid_blocks=2,
                     temporal_up=(True, True, False), z_dim=16, out_ch=3):
    """Convolution FLOPs (2 per multiply-add) of the NEXT-4 VAE decoder for a DiT
    latent grid (F, Ht, Wt): the algorithmic work of the unpadded channel counts, counted per
    stage from the decoder's structure (tests/test_costmodel.py checks it against the oracle's
    executed-conv count)."""
    F, Ht, Wt = grid
    T, H, W = F, 2 * Ht, 2 * Wt

    def conv(t, h, w, cin, cout, taps):
        return 2 * t * h * w * cin * cout * taps

    tot = conv(T, H, W, z_dim, z_dim, 1) + conv(T, H, W, z_dim, dims[0], 27)
    tot += mid_blocks * 2 * conv(T, H, W, dims[0], dims[0], 27)
    cin = dims[0]
    for i in range(4):
        cout = dims[i + 1]
        if i >= 1:
            cin = dims[i] // 2
        for _ in range(blocks):
            tot += conv(T, H, W, cin, cout, 27) + conv(T, H, W, cout, cout, 27)
            if cin != cout:
                tot += conv(T, H, W, cin, cout, 1)
            cin = cout
        if i < 3:
            if temporal_up[i]:
                tot += conv(T - 1, H, W, cout, 2 * cout, 3)
                T = 1 + 2 * (T - 1)
            H, W = 2 * H, 2 * W
            tot += conv(T, H, W, cout, cout // 2, 9)
    return tot + conv(T, H, W, dims[4], out_ch, 27)
