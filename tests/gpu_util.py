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


class LazyBlocks:
    """The L blocks' fp64 parameters generated one layer at a time while the oracle iterates them
    (a 30-layer Wan-1.3B list is ~9 GB in fp64)."""

    def __init__(self, shape):
        self.shape = shape

    def __len__(self):
        return self.shape.layers

    def __iter__(self):
        from synth import models as sm
        for layer in range(self.shape.layers):
            yield sm.as_f64(sm.block_params(self.shape, layer))


def _oracle_one_request(args):
    from oracle import dit
    from synth import models as sm
    shape, z0, grid, step_idx, n_steps, k = args
    glob = sm.as_f64(sm.global_params(shape))
    return dit.dit_steps([z0], [grid], [step_idx], n_steps, k, glob, LazyBlocks(shape), shape.heads)[0]


def oracle_steps_per_request(shape, z0s, grids, step_idx, n_steps, k):
    """oracle dit_steps of a batch, one request per worker process.  Packing is an exact
    re-arrangement of the method (tests/test_oracle_pins.py: the packed oracle equals each request
    alone up to fp64 rounding, <= 1e-12 relative, at block and at step level), so this is the
    batch's oracle result; the workers split the host's cores (numpy's element-wise softmax work
    is single-threaded, BLAS is not)."""
    import multiprocessing as mp
    import os
    n = len(z0s)
    ncpu = len(os.sched_getaffinity(0))
    per = str(max(1, ncpu // n))
    saved = {v: os.environ.get(v) for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS")}
    for v in saved:
        os.environ[v] = per
    try:
        with mp.get_context("spawn").Pool(n) as pool:
            return pool.map(_oracle_one_request,
                            [(shape, np.asarray(z, np.float64), g, i, n_steps, k)
                             for z, g, i in zip(z0s, grids, step_idx)])
    finally:
        for v, val in saved.items():
            if val is None:
                os.environ.pop(v, None)
            else:
                os.environ[v] = val
