"""Counter-based generator (splitmix64) for weights and latent noise.

Definition (SURVEY.md §8(d) "Synthetic inputs"):

    h   = splitmix64(seed XOR (tensor_id << 40) XOR idx)          (uint64, wrapping)
    u   = ((h >> 40) - 2**23) * 2**-23        in [-1, 1), exact in fp32
    w   = RNE_bf16( fp32(u * scale) )          linear weights / biases
    g   = RNE_bf16( fp32(1 + fp32(0.1 * u)) )  RMSNorm gains
    m   = fp32(u * 0.5)                        adaLN modulation tables (fp32)
    z_i = fp32( (u_{4i} + u_{4i+1} + u_{4i+2} + u_{4i+3}) * sqrt(3/4) )   latent noise,
          summed in fp64 (Irwin-Hall(4), unit variance)

splitmix64(x) is Steele/Lea/Flood's SplitMix64 output function applied to
x + 0x9E3779B97F4A7C15 (so splitmix64(0) is the first output of SplitMix64 seeded
with 0: 0xE220A8397B1DCDAF).
"""
import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

# tensor ids (the "tensor_id" field of the counter).  Per-block tensors use
# seed = weight_seed + layer; global tensors use seed = weight_seed + GLOBAL_SEED_OFFSET.
TID = {
    # per block
    "w_qkv": 1, "b_qkv": 2, "g_q": 3, "g_k": 4, "w_o": 5, "b_o": 6,
    "w_1": 7, "b_1": 8, "w_2": 9, "b_2": 10, "mod": 11,
    # global
    "w_pe": 20, "b_pe": 21, "w_t1": 22, "b_t1": 23, "w_t2": 24, "b_t2": 25,
    "w_tp": 26, "b_tp": 27, "mod_head": 28, "w_head": 29, "b_head": 30,
    # per block, text cross-attention (NEXT-1; Wan2.1 block [ext])
    "ln3_w": 12, "ln3_b": 13, "w_cq": 14, "b_cq": 15, "w_ckv": 16, "b_ckv": 17, "g_cq": 18,
    "g_ck": 19, "w_co": 32, "b_co": 33,
    # global, text embedding MLP (text_dim -> D -> D)
    "w_te1": 40, "b_te1": 41, "w_te2": 42, "b_te2": 43,
    # request noise (seed = noise_seed); prompt embeddings (seed = prompt_seed)
    "noise": 0, "prompt_cond": 50, "prompt_uncond": 51,
}
GLOBAL_SEED_OFFSET = 1_000_000


def splitmix64(x):
    """SplitMix64 mix of (x + golden gamma); x: uint64 ndarray."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def uniform_f32(seed, tensor_id, n, offset=0):
    """u[idx] for idx in [offset, offset+n), fp32 in [-1, 1) with 2^-23 resolution."""
    idx = np.arange(offset, offset + n, dtype=np.uint64)
    key = np.uint64(seed) ^ (np.uint64(tensor_id) << np.uint64(40))
    h = splitmix64(key ^ idx)
    top = (h >> np.uint64(40)).astype(np.int64) - (1 << 23)
    return top.astype(np.float32) * np.float32(2.0 ** -23)


def f32_to_bf16_bits(x):
    """Round-to-nearest-even fp32 -> bf16, returned as uint16 bit patterns (no NaN inputs)."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((b >> np.uint64(16)) & np.uint64(1)) + np.uint64(0x7FFF)
    return ((b + r) >> np.uint64(16)).astype(np.uint16)


def bf16_bits_to_f32(bits):
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def bf16_bits_to_f64(bits):
    return bf16_bits_to_f32(bits).astype(np.float64)


def linear_weight_bits(seed, tid, out_f, in_f):
    """Linear weight [out_f, in_f] ~ U(+-sqrt(3/in_f)) -> bf16 bits."""
    scale = np.float32(np.sqrt(3.0 / in_f))
    u = uniform_f32(seed, tid, out_f * in_f)
    return f32_to_bf16_bits(u * scale).reshape(out_f, in_f)


def vector_bf16_bits(seed, tid, n, scale=0.1):
    return f32_to_bf16_bits(uniform_f32(seed, tid, n) * np.float32(scale))


def gain_bf16_bits(seed, tid, n):
    u = uniform_f32(seed, tid, n)
    return f32_to_bf16_bits(np.float32(1.0) + u * np.float32(0.1))


def modulation_f32(seed, tid, rows, cols):
    return (uniform_f32(seed, tid, rows * cols) * np.float32(0.5)).reshape(rows, cols)


def normal_f32(seed, tensor_id, n):
    """n standard-normal fp32 values: Irwin-Hall(4) of the counter uniforms, summed in fp64."""
    u = uniform_f32(seed, tensor_id, 4 * n).astype(np.float64)
    return (u.reshape(-1, 4).sum(axis=1) * np.sqrt(0.75)).astype(np.float32)


def prompt_embeds_bits(prompt_seed, branch, text_len, text_dim):
    """Synthetic text-encoder output [text_len, text_dim] as bf16 bits (branch 0 = cond,
    1 = uncond / negative prompt): RNE_bf16 of standard-normal values."""
    tid = TID["prompt_cond"] if branch == 0 else TID["prompt_uncond"]
    return f32_to_bf16_bits(normal_f32(prompt_seed, tid, text_len * text_dim)).reshape(text_len, text_dim)


def noise_latent_f32(noise_seed, n_tokens, channels=64):
    """Initial latent z_T [n_tokens, channels], token-major, fp32."""
    u = uniform_f32(noise_seed, TID["noise"], 4 * n_tokens * channels).astype(np.float64)
    s = u.reshape(-1, 4).sum(axis=1) * np.sqrt(0.75)
    return s.astype(np.float32).reshape(n_tokens, channels)
