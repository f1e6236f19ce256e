"""NEXT-4 VAE decode on the GPU vs the fp64 oracle (oracle/vae.py): the tcgen05 implicit-GEMM causal
conv (every kernel shape, padding, ragged patches, output modes) and whole decoders; the request
path (decode after the last DiT step) equals decoding the read-back latent bit for bit."""
import numpy as np
import pytest

from oracle import vae as ov
from synth import models as sm
from synth import rng
from synth import vae as sv
from tests.gpu_util import from_dev_bf16, rel_l2, max_row_rel_l2, to_dev_bf16

pytestmark = pytest.mark.gpu
TOL = 1e-2   # BASELINE.json north_star relative-L2 bar (bf16 storage, fp32 accumulation)


@pytest.fixture(scope="module")
def gs():
    import paper_2604_04335_b200 as m
    m.load()
    return m


@pytest.fixture(scope="module")
def ctx(gs):
    c = gs.Context(device=0)
    yield c
    c.close()


def _bf16(g, shape, scale=1.0):
    return rng.f32_to_bf16_bits((g.standard_normal(shape) * scale).astype(np.float32))


@pytest.mark.parametrize("k", [(3, 3, 3), (3, 1, 1), (1, 3, 3), (1, 1, 1)])
@pytest.mark.parametrize("T,H,W,C,Co", [(3, 10, 37, 64, 64), (2, 9, 33, 128, 192), (4, 8, 32, 64, 384),
                                        (1, 5, 70, 128, 256), (2, 17, 31, 192, 128),
                                        # 32-channel K blocks (64B swizzle) and narrow N tiles
                                        (2, 9, 40, 96, 96), (1, 6, 33, 32, 32), (2, 8, 35, 96, 192)])
def test_conv3d_matches_oracle(ctx, T, H, W, C, Co, k):
    import torch
    g = np.random.default_rng(T * 1000 + H * 10 + W + C)
    x = _bf16(g, (T, H, W, C))
    fan = C * k[0] * k[1] * k[2]
    w = _bf16(g, (Co, *k, C), np.sqrt(1.0 / fan))
    b = _bf16(g, (Co,), 0.1)
    out = torch.zeros((T, H, W, Co), dtype=torch.bfloat16, device="cuda")
    ctx.debug_conv3d(to_dev_bf16(x), to_dev_bf16(w), to_dev_bf16(b), out, T, H, W, C, k, Co)
    ref = ov.causal_conv3d(rng.bf16_bits_to_f64(x), rng.bf16_bits_to_f64(w), rng.bf16_bits_to_f64(b))
    got = from_dev_bf16(out)
    assert rel_l2(got, ref) < 4e-3 and max_row_rel_l2(got.reshape(-1, Co), ref.reshape(-1, Co)) < 2e-2


def test_conv3d_residual_interleave_and_clamp_modes(ctx):
    import torch
    g = np.random.default_rng(3)
    T, H, W, C = 3, 6, 40, 64
    x = _bf16(g, (T, H, W, C))
    b = _bf16(g, (2 * C,), 0.1)
    w = _bf16(g, (2 * C, 3, 1, 1, C), np.sqrt(1.0 / (3 * C)))
    xf, wf, bf = (rng.bf16_bits_to_f64(a) for a in (x, w, b))
    # residual epilogue
    r = _bf16(g, (T, H, W, 2 * C))
    out = torch.zeros((T, H, W, 2 * C), dtype=torch.bfloat16, device="cuda")
    ctx.debug_conv3d(to_dev_bf16(x), to_dev_bf16(w), to_dev_bf16(b), out, T, H, W, C, (3, 1, 1), 2 * C,
                     resid=to_dev_bf16(r))
    ref = ov.causal_conv3d(xf, wf, bf) + rng.bf16_bits_to_f64(r)
    assert rel_l2(from_dev_bf16(out), ref) < 4e-3
    # temporal interleave: channel halves of frame t -> output frames 2t+1, 2t+2 (reading V5)
    out2 = torch.zeros((1 + 2 * T, H, W, C), dtype=torch.bfloat16, device="cuda")
    ctx.debug_conv3d(to_dev_bf16(x), to_dev_bf16(w), to_dev_bf16(b), out2, T, H, W, C, (3, 1, 1), 2 * C,
                     out_cs=C, mode=1, out_real=C)
    y = ov.causal_conv3d(xf, wf, bf)
    got = from_dev_bf16(out2)
    for t in range(T):
        assert rel_l2(got[2 * t + 1], y[t, ..., :C]) < 4e-3
        assert rel_l2(got[2 * t + 2], y[t, ..., C:]) < 4e-3
    assert np.all(got[0] == 0)                      # frame 0 untouched by the conv
    # fp32 clamp of the first 3 channels (decoder output, reading V7)
    w3 = _bf16(g, (64, 3, 3, 3, C), 0.2)
    out3 = torch.zeros((T, H, W, 3), dtype=torch.float32, device="cuda")
    ctx.debug_conv3d(to_dev_bf16(x), to_dev_bf16(w3), to_dev_bf16(b[:64]), out3, T, H, W, C, (3, 3, 3), 64,
                     mode=2, out_real=3)
    ref3 = np.clip(ov.causal_conv3d(xf, rng.bf16_bits_to_f64(w3), bf[:64])[..., :3], -1, 1)
    got3 = out3.cpu().numpy().astype(np.float64)
    assert rel_l2(got3, ref3) < 4e-3 and got3.min() >= -1 and got3.max() <= 1


def _decode_case(gs, ctx, shape, grid, seed=5):
    vid = ctx.vae_create(shape.z_dim, shape.dims, shape.blocks, shape.mid_blocks, shape.temporal_up,
                         shape.out_ch, shape.weight_seed)
    g = np.random.default_rng(seed)
    lat = g.standard_normal((int(np.prod(grid)), 64)).astype(np.float32)
    got = ctx.vae_decode(vid, lat, grid, temporal_up=shape.temporal_up, out_ch=shape.out_ch)
    ref = ov.decode(lat.astype(np.float64), grid, sv.vae_params(shape), shape)
    return got, ref


@pytest.mark.parametrize("grid", [(3, 2, 3), (1, 3, 5), (2, 4, 2)])
def test_vae_decode_tiny_matches_oracle(gs, ctx, grid):
    got, ref = _decode_case(gs, ctx, sv.TINY_VAE, grid)
    assert got.shape == ref.shape
    err = rel_l2(got, ref)
    print(f"tiny VAE {grid}: rel-L2 {err:.3e}")
    assert err < TOL


def test_vae_decode_wan_shape_matches_oracle(gs, ctx):
    """The Wan2.1-VAE-shaped decoder (widths 384 / 192 / 96, 96 padded to 128 on the GPU) at a
    small latent grid: 2 latent frames -> 5 video frames of 32 x 48."""
    got, ref = _decode_case(gs, ctx, sv.WAN_VAE, (2, 2, 3))
    err = rel_l2(got, ref)
    print(f"Wan VAE (2,2,3): rel-L2 {err:.3e}")
    assert got.shape == (5, 32, 48, 3) and err < TOL


def test_vae_decode_request_equals_decode_of_latent(gs):
    """The pipeline stage: a request's latent after its DiT steps (SP = 4, sharded) decoded on one
    GPU equals decoding the gathered latent read back to the host, bit for bit."""
    shape = sm.TINY.with_layers(1)
    ctx = gs.Context(device=0, world_size=4, emulated=True)
    mid = ctx.model_create(shape.dim, shape.heads, shape.ffn, shape.layers, shape.weight_seed)
    vs = sv.TINY_VAE
    vid = ctx.vae_create(vs.z_dim, vs.dims, vs.blocks, vs.mid_blocks, vs.temporal_up, vs.out_ch, vs.weight_seed)
    req = ctx.submit(mid, 64, 48, 9, 50, 1000, [0, 1, 2, 3])
    ctx.run_steps([req], [0, 1, 2, 3], 2)
    grid = sm.token_grid(64, 48, 9)
    a = ctx.vae_decode_request(vid, req, grid)
    b = ctx.vae_decode(vid, ctx.read_latent(req), grid, rank=2)
    ctx.close()
    assert a.shape == (9, 48, 64, 3)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


@pytest.mark.slow
def test_vae_decode_fullsize_720p_sampled_windows(gs, ctx):
    """Config 4's latent at full size (DiT grid 21 x 45 x 80 -> 81 x 720 x 1280 x 3, the bench's
    launch configuration) against the oracle on sampled windows.  The decoder is causal in time and
    its spatial receptive field is ~17 latent pixels (conv taps summed over the walk), so the oracle
    decode of a crop -- latent frames 0..1, +-10 tokens around a sample token, clipped at the true
    borders (where the crop's zero padding IS the conv padding) -- equals the full decode on the sample
    token's 16 x 16 output pixels of output frames 0..4 (translation equivariance, pinned in
    tests/test_vae_pins.py)."""
    import torch
    shape = sv.WAN_VAE
    grid = (21, 45, 80)
    vid = ctx.vae_create(shape.z_dim, shape.dims, shape.blocks, shape.mid_blocks, shape.temporal_up,
                         shape.out_ch, shape.weight_seed)
    g = np.random.default_rng(8)
    lat = g.standard_normal((int(np.prod(grid)), 64)).astype(np.float32)
    out = torch.empty(ctx.vae_out_shape(grid), device="cuda", dtype=torch.float32)
    ctx.vae_decode(vid, torch.from_numpy(lat).cuda(), grid, out=out)
    video = out[:5].cpu().numpy().astype(np.float64)            # output frames of latent frames 0, 1
    params = sv.vae_params(shape)
    lat4 = lat.reshape(grid[0], grid[1], grid[2], 64)
    R = 10
    for th, tw in [(22, 40), (0, 0), (44, 79), (3, 77)]:
        h0, h1 = max(0, th - R), min(grid[1], th + R + 1)
        w0, w1 = max(0, tw - R), min(grid[2], tw + R + 1)
        crop = lat4[:2, h0:h1, w0:w1].reshape(-1, 64).astype(np.float64)
        ref = ov.decode(crop, (2, h1 - h0, w1 - w0), params, shape)   # [5, 16 (h1-h0), 16 (w1-w0), 3]
        oh, ow = 16 * (th - h0), 16 * (tw - w0)
        got = video[:, 16 * th:16 * th + 16, 16 * tw:16 * tw + 16]
        want = ref[:, oh:oh + 16, ow:ow + 16]
        err = rel_l2(got, want)
        print(f"720p window at token ({th}, {tw}): rel-L2 {err:.3e}")
        assert err < TOL, (th, tw, err)
