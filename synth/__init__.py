"""Seeded synthetic inputs shared by the oracle side and the GPU side of the tests.

This module holds NO arithmetic of the method (no LayerNorm, attention, GEMM, RoPE,
sampler, ...).  It only defines

* the counter-based generator (splitmix64), which
  `paper_2604_04335_b200/csrc/rng.cu` re-implements independently on the device;
* the model shapes named by BASELINE.json `configs` (+ the SURVEY.md §8 table);
* request token grids (SURVEY.md §8 "Token grids", Wan2.1-VAE-shaped latent).

Everything is plain IEEE arithmetic (integer ops, one fp32 multiply, one fp32->bf16
round-to-nearest-even), so the numpy values and the device values are bitwise equal.
"""
from .rng import (  # noqa: F401
    splitmix64, uniform_f32, f32_to_bf16_bits, bf16_bits_to_f32, bf16_bits_to_f64,
    linear_weight_bits, vector_bf16_bits, gain_bf16_bits, modulation_f32, noise_latent_f32,
    TID,
)
from .models import (  # noqa: F401
    ModelShape, TINY, WAN_1_3B, WAN_14B, MODELS, token_grid, block_params, global_params,
    seq_shards,
)
