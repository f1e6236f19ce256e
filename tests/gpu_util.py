"""Helpers shared by the -m gpu tests (torch is used for device memory only)."""
import numpy as np

from synth import rng


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def max_row_rel_l2(a, b):
    """Largest per-row relative L2 error max_r |a_r - b_r| / |b_r| (rows = tokens), reported beside
    the whole-tensor rel-L2 of the north star."""
    a = np.asarray(a, np.float64).reshape(len(a), -1)
    b = np.asarray(b, np.float64).reshape(len(b), -1)
    return float(np.max(np.linalg.norm(a - b, axis=1) / np.maximum(np.linalg.norm(b, axis=1), 1e-300)))


def bf16_bits(x):
    """fp64/fp32 array -> bf16 bit patterns (RNE)."""
    return rng.f32_to_bf16_bits(np.asarray(x, np.float32))


def to_dev_bf16(bits):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(bits).view(np.int16).copy())
    return t.view(torch.bfloat16).cuda()


def from_dev_bf16(t):
    import torch
    bits = t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
    return rng.bf16_bits_to_f64(bits)


def to_dev(x, dtype):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).to(dtype).cuda()


def randn_bf16(gen, shape, scale=1.0):
    """bf16 bit patterns of N(0, scale^2) samples."""
    return bf16_bits(gen.standard_normal(shape) * scale)
