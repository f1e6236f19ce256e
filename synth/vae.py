"""VAE decoder shape, module walk and seeded parameters (inputs only, no method arithmetic).

SURVEY.md §8(f) NEXT-4: a single-GPU VAE decode stage after the DiT ("the VAE stage always execute[s]
on a single GPU", §4.3).  The paper gives no VAE internals; the shape is Wan2.1-VAE-like
[ext] (DESIGN.md §NEXT-4 readings V1-V8): latent 16 channels, decoder widths (384, 384, 384, 192,
96), 3 residual blocks per stage, temporal upsampling x2 in the first two stages, spatial x2 in the
first three, causal 3-D convolutions, RMS norms over channels, no mid attention (reading V4).

Module walk (the order fixes each module's tensor ids; csrc/vae.cpp builds the same list):
  0 'znorm'                  latent de-normalisation: mean (slot 0), std (slot 1), fp32 [16]
  1 'post'  conv 1x1x1 16->16
  2 'conv_in' conv 3x3x3 16->384
  then residual blocks (norm1, conv1 3x3x3, norm2, conv2 3x3x3, [skip 1x1x1 when cin != cout]):
    2 mid blocks 384->384; stage 0: 3 x 384->384, upsample3d(384); stage 1: 192->384, 2 x 384->384,
    upsample3d(384); stage 2: 3 x 192->192, upsample2d(192); stage 3: 3 x 96->96
  upsample3d(C): 'tconv' conv 3x1x1 C->2C, then 'sconv' conv 1x3x3 C->C/2 after nearest x2 in H, W
  upsample2d(C): 'sconv' conv 1x3x3 C->C/2 after nearest x2
  'norm_out' (gamma), 'conv_out' conv 3x3x3 96->3.
Tensor ids: tid = 200 + 4 * module_index + slot (slot 0 weight / gamma / mean, 1 bias / std);
seed = weight_seed.  Conv weights [Cout, kt, kh, kw, Cin] ~ U(+-sqrt(3 / (Cin kt kh kw))) -> bf16;
biases U(+-0.1) -> bf16; gammas 1 + U(+-0.1) -> bf16; mean U(+-0.5), std 1 + 0.25 U fp32.
"""
from dataclasses import dataclass

import numpy as np

from .rng import f32_to_bf16_bits, uniform_f32


@dataclass(frozen=True)
class VaeShape:
    name: str = "wan-vae-dec"
    z_dim: int = 16
    dims: tuple = (384, 384, 384, 192, 96)
    blocks: int = 3                     # residual blocks per up stage (Wan num_res_blocks + 1)
    mid_blocks: int = 2
    temporal_up: tuple = (True, True, False)
    out_ch: int = 3
    weight_seed: int = 4321


WAN_VAE = VaeShape()
# a narrow variant with the same walk (tests at small sizes)
TINY_VAE = VaeShape("tiny-vae-dec", dims=(128, 128, 128, 128, 64), weight_seed=77)


def vae_modules(shape: VaeShape):
    """[(name, kind, cin, cout, (kt, kh, kw))] in walk order; kind in {znorm, conv, norm}."""
    mods = [("znorm", "znorm", shape.z_dim, shape.z_dim, None),
            ("post", "conv", shape.z_dim, shape.z_dim, (1, 1, 1)),
            ("conv_in", "conv", shape.z_dim, shape.dims[0], (3, 3, 3))]

    def res(prefix, cin, cout):
        mods.extend([(prefix + ".norm1", "norm", cin, cin, None),
                     (prefix + ".conv1", "conv", cin, cout, (3, 3, 3)),
                     (prefix + ".norm2", "norm", cout, cout, None),
                     (prefix + ".conv2", "conv", cout, cout, (3, 3, 3))])
        if cin != cout:
            mods.append((prefix + ".skip", "conv", cin, cout, (1, 1, 1)))

    d = shape.dims
    for b in range(shape.mid_blocks):
        res(f"mid.{b}", d[0], d[0])
    cin = d[0]
    nst = len(d) - 1
    for i in range(nst):
        cout = d[i + 1]
        if i >= 1:
            cin = d[i] // 2
        for b in range(shape.blocks):
            res(f"up{i}.{b}", cin, cout)
            cin = cout
        if i < nst - 1:
            if shape.temporal_up[i]:
                mods.append((f"up{i}.tconv", "conv", cout, 2 * cout, (3, 1, 1)))
            mods.append((f"up{i}.sconv", "conv", cout, cout // 2, (1, 3, 3)))
    mods.append(("norm_out", "norm", d[-1], d[-1], None))
    mods.append(("conv_out", "conv", d[-1], shape.out_ch, (3, 3, 3)))
    return mods


def vae_params(shape: VaeShape):
    """{module name: {tensor: array}}; bf16 tensors as uint16 bits, fp32 as float32."""
    s = shape.weight_seed
    out = {}
    for m, (name, kind, cin, cout, k) in enumerate(vae_modules(shape)):
        tid = 200 + 4 * m
        if kind == "znorm":
            out[name] = {"mean": uniform_f32(s, tid, cin) * np.float32(0.5),
                         "std": np.float32(1.0) + uniform_f32(s, tid + 1, cin) * np.float32(0.25)}
        elif kind == "norm":
            out[name] = {"gamma": f32_to_bf16_bits(np.float32(1.0) + np.float32(0.1) * uniform_f32(s, tid, cin))}
        else:
            kt, kh, kw = k
            fan = cin * kt * kh * kw
            scale = np.float32(np.sqrt(3.0 / fan))
            w = f32_to_bf16_bits(uniform_f32(s, tid, cout * fan) * scale).reshape(cout, kt, kh, kw, cin)
            b = f32_to_bf16_bits(uniform_f32(s, tid + 1, cout) * np.float32(0.1))
            out[name] = {"w": w, "b": b}
    return out


def output_frames(frames_lat, shape: VaeShape = WAN_VAE):
    """Frames decoded from F_lat latent frames: each temporal x2 stage maps T -> 1 + 2 (T - 1)."""
    t = frames_lat
    for up in shape.temporal_up:
        if up:
            t = 1 + 2 * (t - 1)
    return t
