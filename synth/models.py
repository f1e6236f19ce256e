"""Model shapes, token grids and seeded parameter sets (inputs only, no method arithmetic).

Shapes: BASELINE.json `configs` + SURVEY.md §8 shape table (F, L from public Wan2.1
configs, marked [ext] there).  Token grid: SURVEY.md §8 "Token grids" — Wan2.1-VAE
stride (4, 8, 8), patch (1, 2, 2): n = F_lat * (h/16) * (w/16), F_lat = 1 + (frames-1)/4,
64 latent floats per token.
"""
from dataclasses import dataclass, replace

import numpy as np

from .rng import (GLOBAL_SEED_OFFSET, TID, gain_bf16_bits, linear_weight_bits, modulation_f32,
                  prompt_embeds_bits, vector_bf16_bits)


@dataclass(frozen=True)
class ModelShape:
    name: str
    dim: int
    heads: int
    ffn: int
    layers: int
    lat: int = 64            # P_lat = C * pt * ph * pw = 16 * 1 * 2 * 2
    freq_dim: int = 256      # sinusoidal time-embedding width (Wan [ext])
    weight_seed: int = 1234
    cross_attn: bool = False  # NEXT-1: text cross-attention in every block (Wan2.1 [ext])
    text_len: int = 512       # umT5 context length (Wan [ext])
    text_dim: int = 4096      # umT5 width (Wan [ext])

    @property
    def head_dim(self):
        return self.dim // self.heads

    def with_layers(self, layers):
        return replace(self, layers=layers)

    def with_text(self, text_len=512, text_dim=4096):
        return replace(self, cross_attn=True, text_len=text_len, text_dim=text_dim)


TINY = ModelShape("tiny", 384, 6, 1536, 1)
WAN_1_3B = ModelShape("wan-1.3b", 1536, 12, 8960, 30)
WAN_14B = ModelShape("wan-14b", 5120, 40, 13824, 40)
MODELS = {m.name: m for m in (TINY, WAN_1_3B, WAN_14B)}


def token_grid(width, height, frames=1):
    """(F_lat, H_t, W_t) token grid of a request (SURVEY.md §8 'Token grids')."""
    if width % 16 or height % 16 or (frames - 1) % 4:
        raise ValueError("width/height must be multiples of 16 and frames = 1 mod 4")
    return (1 + (frames - 1) // 4, height // 16, width // 16)


def seq_shards(n, p):
    """Contiguous token shard bounds of n tokens over p ranks (SURVEY.md §8(c) reading 10)."""
    return [((i * n) // p, ((i + 1) * n) // p) for i in range(p)]


def block_params(shape: ModelShape, layer: int):
    """Seeded parameters of block `layer`. bf16 tensors are uint16 bit patterns."""
    s = shape.weight_seed + layer
    D, F = shape.dim, shape.ffn
    return {
        "w_qkv": linear_weight_bits(s, TID["w_qkv"], 3 * D, D),
        "b_qkv": vector_bf16_bits(s, TID["b_qkv"], 3 * D),
        "g_q": gain_bf16_bits(s, TID["g_q"], D),
        "g_k": gain_bf16_bits(s, TID["g_k"], D),
        "w_o": linear_weight_bits(s, TID["w_o"], D, D),
        "b_o": vector_bf16_bits(s, TID["b_o"], D),
        "w_1": linear_weight_bits(s, TID["w_1"], F, D),
        "b_1": vector_bf16_bits(s, TID["b_1"], F),
        "w_2": linear_weight_bits(s, TID["w_2"], D, F),
        "b_2": vector_bf16_bits(s, TID["b_2"], D),
        "mod": modulation_f32(s, TID["mod"], 6, D),
        **(cross_block_params(shape, layer) if shape.cross_attn else {}),
    }


def cross_block_params(shape: ModelShape, layer: int):
    """Text cross-attention tensors of block `layer` (NEXT-1)."""
    s = shape.weight_seed + layer
    D = shape.dim
    return {
        "ln3_w": gain_bf16_bits(s, TID["ln3_w"], D),
        "ln3_b": vector_bf16_bits(s, TID["ln3_b"], D),
        "w_cq": linear_weight_bits(s, TID["w_cq"], D, D),
        "b_cq": vector_bf16_bits(s, TID["b_cq"], D),
        "w_ckv": linear_weight_bits(s, TID["w_ckv"], 2 * D, D),
        "b_ckv": vector_bf16_bits(s, TID["b_ckv"], 2 * D),
        "g_cq": gain_bf16_bits(s, TID["g_cq"], D),
        "g_ck": gain_bf16_bits(s, TID["g_ck"], D),
        "w_co": linear_weight_bits(s, TID["w_co"], D, D),
        "b_co": vector_bf16_bits(s, TID["b_co"], D),
    }


def prompt_embeds(shape: ModelShape, prompt_seed: int, branch: int):
    """Synthetic prompt embeddings [text_len, text_dim] (bf16 bits) of one CFG branch."""
    return prompt_embeds_bits(prompt_seed, branch, shape.text_len, shape.text_dim)


def global_params(shape: ModelShape):
    s = shape.weight_seed + GLOBAL_SEED_OFFSET
    D, P, T = shape.dim, shape.lat, shape.freq_dim
    return {
        "w_pe": linear_weight_bits(s, TID["w_pe"], D, P),
        "b_pe": vector_bf16_bits(s, TID["b_pe"], D),
        "w_t1": linear_weight_bits(s, TID["w_t1"], D, T),
        "b_t1": vector_bf16_bits(s, TID["b_t1"], D),
        "w_t2": linear_weight_bits(s, TID["w_t2"], D, D),
        "b_t2": vector_bf16_bits(s, TID["b_t2"], D),
        "w_tp": linear_weight_bits(s, TID["w_tp"], 6 * D, D),
        "b_tp": vector_bf16_bits(s, TID["b_tp"], 6 * D),
        "mod_head": modulation_f32(s, TID["mod_head"], 2, D),
        "w_head": linear_weight_bits(s, TID["w_head"], P, D),
        "b_head": vector_bf16_bits(s, TID["b_head"], P),
        **({"w_te1": linear_weight_bits(s, TID["w_te1"], D, shape.text_dim),
            "b_te1": vector_bf16_bits(s, TID["b_te1"], D),
            "w_te2": linear_weight_bits(s, TID["w_te2"], D, D),
            "b_te2": vector_bf16_bits(s, TID["b_te2"], D)} if shape.cross_attn else {}),
    }


def as_f64(params):
    """Exact upcast of a parameter dict (bf16 bits or fp32) to fp64 arrays."""
    from .rng import bf16_bits_to_f64
    out = {}
    for k, v in params.items():
        out[k] = bf16_bits_to_f64(v) if v.dtype == np.uint16 else v.astype(np.float64)
    return out
