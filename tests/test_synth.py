"""Pins for the seeded input generator (synth/): splitmix64 test vectors, bf16 RNE, shapes."""
import numpy as np

from synth import models as sm
from synth import rng


def test_splitmix64_reference_vectors():
    # SplitMix64 seeded with 0: first outputs (Vigna's reference splitmix64.c)
    assert int(rng.splitmix64(np.array([0], np.uint64))[0]) == 0xE220A8397B1DCDAF
    g = 0x9E3779B97F4A7C15
    assert int(rng.splitmix64(np.array([g], np.uint64))[0]) == 0x6E789E6AA1B965F4
    assert int(rng.splitmix64(np.array([(2 * g) & (2**64 - 1)], np.uint64))[0]) == 0x06C45D188009454F


def test_uniform_range_and_resolution():
    u = rng.uniform_f32(7, 3, 1 << 16)
    assert u.dtype == np.float32
    assert u.min() >= -1.0 and u.max() < 1.0
    assert np.all((u.astype(np.float64) * 2**23) == np.round(u.astype(np.float64) * 2**23))
    assert abs(float(u.mean())) < 0.01 and abs(float(u.var()) - 1 / 3) < 0.01


def test_bf16_rne():
    x = np.array([1.0, 1.0 + 2**-8, 1.0 + 3 * 2**-8, 1.0 + 2**-8 + 2**-20, -2.5, 0.0],
                 dtype=np.float32)
    bits = rng.f32_to_bf16_bits(x)
    back = rng.bf16_bits_to_f32(bits)
    # 1+2^-8 is a tie -> even (1.0); 1+3*2^-8 tie -> 1+2^-6... (even mantissa); above tie -> up
    assert back[0] == 1.0
    assert back[1] == 1.0
    assert back[2] == np.float32(1.0 + 4 * 2**-8)
    assert back[3] == np.float32(1.0 + 2**-7)
    assert back[4] == -2.5 and back[5] == 0.0


def test_noise_unit_variance():
    z = rng.noise_latent_f32(1000, 4096)
    assert z.shape == (4096, 64) and z.dtype == np.float32
    assert abs(float(z.mean())) < 0.01 and abs(float(z.std()) - 1.0) < 0.01


def test_token_grids_match_baseline_counts():
    assert np.prod(sm.token_grid(256, 256)) == 256
    assert np.prod(sm.token_grid(1024, 1024)) == 4096
    assert np.prod(sm.token_grid(832, 480, 81)) == 32760
    assert np.prod(sm.token_grid(1280, 720, 81)) == 75600


def test_seq_shards_cover():
    for n in (1, 7, 32760, 75600):
        for p in (1, 2, 4, 8):
            sh = sm.seq_shards(n, p)
            assert sh[0][0] == 0 and sh[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(sh, sh[1:]))


def test_param_shapes_and_determinism():
    shape = sm.ModelShape("t", 64, 2, 128, 1)
    p1 = sm.block_params(shape, 0)
    p2 = sm.block_params(shape, 0)
    assert p1["w_qkv"].shape == (192, 64) and p1["w_qkv"].dtype == np.uint16
    assert p1["mod"].dtype == np.float32
    for k in p1:
        np.testing.assert_array_equal(p1[k], p2[k])
    assert not np.array_equal(sm.block_params(shape, 1)["w_o"], p1["w_o"])
