"""Pin P1: the paper's own cost model (Tab. arithmetic_intensity)."""
import os

import pytest

from paper_2604_04335_b200 import costmodel

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "tab3_arithmetic_intensity.txt")


def _rows():
    for line in open(GOLDEN):
        if line.startswith("#") or not line.strip():
            continue
        m, L, D, F, N, fl, ai = line.split()
        yield m, int(L), int(D), int(F), int(N), float(fl), float(ai)


@pytest.mark.parametrize("row", list(_rows()), ids=lambda r: f"{r[0]}-{r[4]}")
def test_tab3_flops_and_ai(row):
    _m, L, D, F, N, flops_t, ai = row
    fl = costmodel.paper_flops_per_step(L, N, D, F)
    by = costmodel.paper_bytes_per_step(L, N, D, F)
    # printed to 2 decimals (T) and to the integer (FLOP/B)
    assert abs(fl / 1e12 - flops_t) <= 0.006
    assert abs(fl / by - ai) <= 0.6


def test_block_split_matches_step_model():
    # flops_per_block summed over L single-request blocks == the paper's per-step formula
    L, D, F, N = 30, 3072, 14336, 12096
    assert L * costmodel.flops_per_block([N], D, F) == costmodel.paper_flops_per_step(L, N, D, F)
    # varlen: attention term is sum n^2 (block diagonal), GEMM term is linear in N
    assert costmodel.attn_flops_per_block([3, 4], 8) == 4 * 8 * (9 + 16)


def test_vae_decode_flops_matches_oracle_walk():
    """bench.py's VAE work count (costmodel, product side) equals the oracle's count of the convs
    it executes (oracle/vae.py decode_flops, pinned in tests/test_vae_pins.py) -- two independent
    walks of the decoder."""
    from oracle import vae as ov
    from paper_2604_04335_b200 import costmodel
    from synth import vae as sv
    for shape in (sv.WAN_VAE, sv.TINY_VAE):
        for grid in [(21, 45, 80), (1, 64, 64), (3, 2, 3)]:
            assert costmodel.vae_decode_flops(grid, shape.dims, shape.blocks, shape.mid_blocks,
                                              shape.temporal_up, shape.z_dim, shape.out_ch) == \
                ov.decode_flops(grid, shape, sv.vae_modules)
