"""GenServe DiT-step hot path on B200 (sm_100a): thin ctypes binding over libgs.so.

Argument marshalling only — every step of the path runs in the CUDA kernels of
`csrc/` behind the C-ABI declared in `include/gs.h`.  There is no CPU fallback: if
libgs.so is missing or fails to load, `load()` raises.
"""
import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgs.so")

GS_OK, GS_EINVAL, GS_ESTATE, GS_ENOMEM, GS_ECUDA, GS_ENCCL, GS_EUNSUPPORTED = 0, -1, -2, -3, -4, -5, -6
REQ_PLACED, REQ_RUNNING, REQ_PAUSED, REQ_DONE, REQ_QUEUED = 0, 1, 2, 3, 4
EPI_BF16, EPI_GELU_BF16, EPI_F32, EPI_RESID_F32, EPI_EULER_F32 = 0, 1, 2, 3, 4


class GsError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"gs error {code}: {msg}")
        self.code = code


class ModelDesc(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int), ("heads", ctypes.c_int), ("ffn", ctypes.c_int),
                ("layers", ctypes.c_int), ("lat", ctypes.c_int), ("freq_dim", ctypes.c_int),
                ("rope_theta", ctypes.c_float), ("eps", ctypes.c_float),
                ("flow_shift", ctypes.c_float), ("weight_seed", ctypes.c_uint64),
                ("cross_attn", ctypes.c_int), ("text_len", ctypes.c_int), ("text_dim", ctypes.c_int)]


class VaeDesc(ctypes.Structure):
    """gs_vae_desc (include/gs.h): the VAE decoder shape (synth/vae.py VaeShape)."""
    _fields_ = [("z_dim", ctypes.c_int), ("dims", ctypes.c_int * 5), ("blocks", ctypes.c_int),
                ("mid_blocks", ctypes.c_int), ("temporal_up", ctypes.c_int * 3), ("out_ch", ctypes.c_int),
                ("weight_seed", ctypes.c_uint64)]


class Xfer(ctypes.Structure):
    """gs_xfer (include/gs.h): one transfer of an exchange plan."""
    _fields_ = [("op", ctypes.c_int), ("peer", ctypes.c_int), ("src_buf", ctypes.c_int),
                ("dst_buf", ctypes.c_int), ("src_off", ctypes.c_longlong),
                ("dst_off", ctypes.c_longlong), ("rows", ctypes.c_longlong),
                ("width", ctypes.c_longlong), ("src_pitch", ctypes.c_longlong),
                ("dst_pitch", ctypes.c_longlong)]


XFER_SEND, XFER_RECV, XFER_COPY = 0, 1, 2
BUF_SEND, BUF_RECV, BUF_O, BUF_STAGE, BUF_ORECV, BUF_OLD, BUF_NEW = range(7)

_P = ctypes.c_void_p
_I = ctypes.c_int
_IP = ctypes.POINTER(ctypes.c_int)
_FP = ctypes.POINTER(ctypes.c_float)
_U64 = ctypes.c_uint64
_SIG = {
    "gs_nccl_unique_id": [_P],
    "gs_init": [_I, _I, _I, _P, ctypes.POINTER(_P)],
    "gs_init_emulated": [_I, _I, ctypes.POINTER(_P)],
    "gs_destroy": [_P],
    "gs_last_error": [_P],
    "gs_info": [_P, _IP, _IP, _IP],
    "gs_model_create": [_P, ctypes.POINTER(ModelDesc), _IP],
    "gs_get_weight": [_P, _I, _I, ctypes.c_char_p, _P, ctypes.c_size_t],
    "gs_submit": [_P, _I, _I, _I, _I, _I, _U64, _FP, _IP, _I, ctypes.POINTER(_U64)],
    "gs_submit_text": [_P, _I, _I, _I, _I, _I, _U64, _U64, ctypes.c_float, _FP, _P, _IP, _I,
                       ctypes.POINTER(_U64)],
    "gs_run_steps": [_P, ctypes.POINTER(_U64), _I, _IP, _I, _I, _IP],
    "gs_run_steps_async": [_P, ctypes.POINTER(_U64), _I, _IP, _I, _I, ctypes.POINTER(_U64)],
    "gs_wait": [_P, _U64, _IP],
    "gs_ticket_done": [_P, _U64],
    "gs_place": [_P, _U64, _IP, _I],
    "gs_preempt": [_P, _U64, _IP],
    "gs_resume": [_P, _U64, _IP, _I],
    "gs_query": [_P, _U64, _IP, _IP, _IP, _IP, _IP, _IP],
    "gs_read_latent": [_P, _U64, _FP, ctypes.c_size_t],
    "gs_release": [_P, _U64],
    "gs_profile": [_P, _I, _I],
    "gs_stats": [_P, ctypes.c_char_p, ctypes.c_size_t],
    "gs_stream": [_P, _I, ctypes.POINTER(_P)],
    "gs_debug_gemm": [_P, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _I, _P, _FP],
    "gs_debug_gemm_ssq": [_P, _I, _I, _I, _P, _P, _P, _P, _P, _I],
    "gs_debug_attention": [_P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _IP, _IP, _I],
    "gs_debug_block": [_P, _I, _I, _FP, _I, _IP, _IP, _IP, _FP, _P],
    "gs_debug_time_embed": [_P, _I, _I, _FP, _FP, _FP],
    "gs_debug_attention_trace": [_P, ctypes.c_size_t],
    "gs_debug_attention_ctatime": [_P, ctypes.c_size_t],
    "gs_plan_a2a": [_I, _I, _I, _I, _IP, _I, _I, ctypes.POINTER(Xfer), _I, _IP,
                    ctypes.POINTER(ctypes.c_longlong)],
    "gs_plan_a2a_usp": [_I, _I, _I, _I, _I, _IP, _I, _I, ctypes.POINTER(Xfer), _I, _IP,
                        ctypes.POINTER(ctypes.c_longlong)],
    "gs_plan_reshard": [_I, _I, _IP, _I, _IP, _I, _I, ctypes.POINTER(Xfer), _I, _IP],
    "gs_plan_peer": [_I, _I, _I, _IP, _I, _I, ctypes.POINTER(ctypes.c_longlong), _IP,
                     ctypes.POINTER(ctypes.c_longlong)],
    "gs_set_option": [_P, ctypes.c_char_p, ctypes.c_longlong],
    "gs_vae_create": [_P, ctypes.POINTER(VaeDesc), _IP],
    "gs_vae_decode": [_P, _I, _I, _P, _I, _I, _I, _P, _I],
    "gs_vae_decode_request": [_P, _I, _U64, _P],
    "gs_debug_conv3d": [_P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _I, _I, _I, _I],
}
_lib = None


def load(path=LIB_PATH):
    """Load libgs.so (raises if absent — the product path has no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("GS_LIB", path)  # A/B runs against another build (tools/*_ab.sh)
    if not os.path.exists(path):
        raise RuntimeError(f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    for name, args in _SIG.items():
        fn = getattr(lib, name, None)
        if fn is None:  # an older libgs.so loaded for an A/B comparison (tools/kbench.py --lib)
            continue
        fn.argtypes = args
        fn.restype = ctypes.c_char_p if name == "gs_last_error" else (None if name == "gs_destroy" else ctypes.c_int)
    _lib = lib
    return lib


def _ints(xs):
    arr = (ctypes.c_int * max(len(xs), 1))(*xs)
    return arr


def _fl(xs):
    return (ctypes.c_float * max(len(xs), 1))(*xs)


def _ptr(x):
    """Device pointer of a torch tensor (or int / None)."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    return x.data_ptr()


def nccl_unique_id():
    buf = ctypes.create_string_buffer(128)
    rc = load().gs_nccl_unique_id(buf)
    if rc != GS_OK:
        raise GsError(rc, "ncclGetUniqueId failed")
    return buf.raw


def _xfers(call):
    n = ctypes.c_int()
    rc = call(None, 0, ctypes.byref(n))
    if rc != GS_OK:
        raise GsError(rc, "plan arguments rejected")
    arr = (Xfer * max(n.value, 1))()
    rc = call(arr, n.value, ctypes.byref(n))
    if rc != GS_OK:
        raise GsError(rc, "plan failed")
    return [{f: getattr(arr[i], f) for f, _t in Xfer._fields_} for i in range(n.value)]


def plan_a2a(kind, p, me, n_tokens, heads, head_dim, ring=1):
    """Host-only Ulysses exchange plan of SP position `me` (kind 0: K/V seq->head, 2: Q, 1: O
    head->seq); ring > 1 = the USP hybrid's partition (gs_plan_a2a_usp).  Returns (list of transfer
    dicts, staging elements)."""
    lib = load()
    stage = ctypes.c_longlong()
    xs = _xfers(lambda out, mx, n: lib.gs_plan_a2a_usp(kind, p, ring, me, len(n_tokens), _ints(n_tokens),
                                                       heads, head_dim, out, mx, n, ctypes.byref(stage)))
    return xs, stage.value


def plan_reshard(n_tokens, lat, old_ranks, new_ranks, me):
    """Host-only latent re-shard plan of global rank `me`."""
    lib = load()
    return _xfers(lambda out, mx, n: lib.gs_plan_reshard(n_tokens, lat, _ints(old_ranks),
                                                         len(old_ranks), _ints(new_ranks),
                                                         len(new_ranks), me, out, mx, n))


def plan_peer(p, me, n_tokens, heads, head_dim):
    """Peer-store addressing of the fused all-to-alls for SP position `me` (include/gs.h
    gs_plan_peer): (row_delta [nreq], own_lo [nreq, p], o_base [nreq, p]); raises GsError
    (GS_EUNSUPPORTED) when p does not divide heads."""
    lib = load()
    B = len(n_tokens)
    rd = (ctypes.c_longlong * B)()
    ol = (ctypes.c_int * (B * p))()
    ob = (ctypes.c_longlong * (B * p))()
    rc = lib.gs_plan_peer(p, me, B, _ints(n_tokens), heads, head_dim, rd, ol, ob)
    if rc != GS_OK:
        raise GsError(rc, "gs_plan_peer rejected its arguments")
    return (np.array(rd[:], dtype=np.int64), np.array(ol[:], dtype=np.int64).reshape(B, p),
            np.array(ob[:], dtype=np.int64).reshape(B, p))


class Context:
    """One process-side context: a CUDA device and its ranks (see include/gs.h)."""

    def __init__(self, device=0, world_size=1, rank=0, nccl_uid=None, emulated=False):
        lib = load()
        self._lib = lib
        h = ctypes.c_void_p()
        if emulated:
            rc = lib.gs_init_emulated(device, world_size, ctypes.byref(h))
        else:
            rc = lib.gs_init(device, world_size, rank, nccl_uid, ctypes.byref(h))
        self._h = h
        if rc != GS_OK:
            msg = lib.gs_last_error(h).decode() if h.value else "init failed"
            raise GsError(rc, msg)
        self.world_size = world_size
        self.rank = rank
        self.emulated = emulated

    def _ck(self, rc):
        if rc != GS_OK:
            raise GsError(rc, self._lib.gs_last_error(self._h).decode())
        return rc

    def close(self):
        if self._h and self._h.value:
            self._lib.gs_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_option(self, key, value):
        """Runtime option (include/gs.h gs_set_option), e.g. ("a2a", 0 | 1)."""
        self._ck(self._lib.gs_set_option(self._h, key.encode(), int(value)))

    def info(self):
        a, b, c = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        self._ck(self._lib.gs_info(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
        return {"num_sms": a.value, "world_size": b.value, "nlocal": c.value}

    # ---------------------------------------------------------------- models
    def model_create(self, dim, heads, ffn, layers, weight_seed=1234, lat=64, freq_dim=256,
                     rope_theta=10000.0, eps=1e-6, flow_shift=5.0, cross_attn=False, text_len=512,
                     text_dim=4096):
        d = ModelDesc(dim, heads, ffn, layers, lat, freq_dim, rope_theta, eps, flow_shift, weight_seed,
                      int(cross_attn), text_len, text_dim)
        mid = ctypes.c_int()
        self._ck(self._lib.gs_model_create(self._h, ctypes.byref(d), ctypes.byref(mid)))
        return mid.value

    def get_weight(self, model, layer, name, shape, dtype):
        out = np.empty(shape, dtype=dtype)
        self._ck(self._lib.gs_get_weight(self._h, model, layer, name.encode(),
                                         out.ctypes.data_as(ctypes.c_void_p), out.nbytes))
        return out

    # ---------------------------------------------------------------- requests
    @staticmethod
    def _n_tokens(width, height, frames):
        return (1 + (frames - 1) // 4) * (height // 16) * (width // 16)

    def _latent_arg(self, init_latent, width, height, frames, lat=64):
        """The caller's initial latent as a float32 [n_tokens * lat] buffer (size checked here:
        the C side reads exactly that many floats)."""
        if init_latent is None:
            return None, None
        arr = np.ascontiguousarray(init_latent, dtype=np.float32)
        n = self._n_tokens(width, height, frames)
        if arr.size != n * lat:
            raise ValueError(f"init_latent has {arr.size} floats, the request needs {n} x {lat}")
        return arr, arr.ctypes.data_as(_FP)

    def _ranks_arg(self, ranks):
        """ranks=None submits a QUEUED request (placed later with place())."""
        if ranks is None:
            return None, 0
        return _ints(ranks), len(ranks)

    def submit(self, model, width, height, frames, steps, noise_seed, ranks, init_latent=None):
        rid = ctypes.c_uint64()
        keep, lat = self._latent_arg(init_latent, width, height, frames)
        rk, nr = self._ranks_arg(ranks)
        self._ck(self._lib.gs_submit(self._h, model, width, height, frames, steps, noise_seed, lat,
                                     rk, nr, ctypes.byref(rid)))
        del keep
        return rid.value

    def submit_text(self, model, width, height, frames, steps, noise_seed, ranks, prompt_seed=0,
                    cfg_scale=0.0, prompt_embeds=None, init_latent=None, text_len=None, text_dim=None):
        """Cross-attention models: prompt_embeds = uint16 (bf16 bits) [nb, text_len, text_dim] or
        None for the synthetic prompt of prompt_seed; cfg_scale > 0 enables CFG (nb = 2).  The
        prompt's shape is checked against nb (and text_len / text_dim when given)."""
        rid = ctypes.c_uint64()
        keep, lat = self._latent_arg(init_latent, width, height, frames)
        pe = None
        if prompt_embeds is not None:
            prompt_embeds = np.ascontiguousarray(prompt_embeds, dtype=np.uint16)
            nb = 2 if cfg_scale > 0 else 1
            if prompt_embeds.ndim != 3 or prompt_embeds.shape[0] != nb:
                raise ValueError(f"prompt_embeds must be [{nb}, text_len, text_dim] (cfg_scale={cfg_scale})")
            if (text_len is not None and prompt_embeds.shape[1] != text_len) or \
                    (text_dim is not None and prompt_embeds.shape[2] != text_dim):
                raise ValueError(f"prompt_embeds shape {prompt_embeds.shape} != [{nb}, {text_len}, {text_dim}]")
            pe = prompt_embeds.ctypes.data_as(ctypes.c_void_p)
        rk, nr = self._ranks_arg(ranks)
        self._ck(self._lib.gs_submit_text(self._h, model, width, height, frames, steps, noise_seed,
                                          prompt_seed, cfg_scale, lat, pe, rk, nr, ctypes.byref(rid)))
        del keep
        return rid.value

    def place(self, req, ranks):
        """First placement of a QUEUED request (include/gs.h gs_place)."""
        self._ck(self._lib.gs_place(self._h, req, _ints(ranks), len(ranks)))

    def run_steps(self, reqs, ranks, k):
        ids = (ctypes.c_uint64 * len(reqs))(*reqs)
        done = ctypes.c_int()
        self._ck(self._lib.gs_run_steps(self._h, ids, len(reqs), _ints(ranks), len(ranks), k,
                                        ctypes.byref(done)))
        return done.value

    def run_steps_async(self, reqs, ranks, k):
        """Start k steps on a worker thread of the context; returns a ticket for wait()."""
        ids = (ctypes.c_uint64 * len(reqs))(*reqs)
        t = ctypes.c_uint64()
        self._ck(self._lib.gs_run_steps_async(self._h, ids, len(reqs), _ints(ranks), len(ranks), k,
                                              ctypes.byref(t)))
        return t.value

    def wait(self, ticket):
        """Wait for an asynchronous run; returns the steps it ran (raises its error)."""
        done = ctypes.c_int()
        self._ck(self._lib.gs_wait(self._h, ticket, ctypes.byref(done)))
        return done.value

    def ticket_done(self, ticket):
        rc = self._lib.gs_ticket_done(self._h, ticket)
        if rc < 0:
            self._ck(rc)
        return bool(rc)

    def preempt(self, req):
        s = ctypes.c_int()
        self._ck(self._lib.gs_preempt(self._h, req, ctypes.byref(s)))
        return s.value

    def resume(self, req, ranks):
        self._ck(self._lib.gs_resume(self._h, req, _ints(ranks), len(ranks)))

    def query(self, req):
        v = [ctypes.c_int() for _ in range(5)]
        ranks = (ctypes.c_int * 8)()
        self._ck(self._lib.gs_query(self._h, req, ctypes.byref(v[0]), ctypes.byref(v[1]),
                                    ctypes.byref(v[2]), ranks, ctypes.byref(v[3]),
                                    ctypes.byref(v[4])))
        return {"steps_done": v[0].value, "steps_total": v[1].value,
                "ranks": list(ranks[:v[2].value]), "state": v[3].value, "n_tokens": v[4].value}

    def read_latent(self, req, n_tokens=None, lat=64, out=None):
        """Gather the request's latent [n_tokens, lat] fp32 into `out` (e.g. a pinned host buffer)
        or a new array."""
        if n_tokens is None:
            n_tokens = self.query(req)["n_tokens"]
        if out is None:
            out = np.zeros((n_tokens, lat), dtype=np.float32)
        elif out.dtype != np.float32 or not out.flags.c_contiguous or out.size != n_tokens * lat:
            raise ValueError("out must be a C-contiguous float32 array of n_tokens * lat elements")
        self._ck(self._lib.gs_read_latent(self._h, req, out.ctypes.data_as(_FP), out.size))
        return out

    def release(self, req):
        self._ck(self._lib.gs_release(self._h, req))

    # ---------------------------------------------------------------- VAE decode (NEXT-4)
    def vae_create(self, z_dim=16, dims=(384, 384, 384, 192, 96), blocks=3, mid_blocks=2,
                   temporal_up=(True, True, False), out_ch=3, weight_seed=4321):
        d = VaeDesc(z_dim, (ctypes.c_int * 5)(*dims), blocks, mid_blocks,
                    (ctypes.c_int * 3)(*[int(x) for x in temporal_up]), out_ch, weight_seed)
        vid = ctypes.c_int()
        self._ck(self._lib.gs_vae_create(self._h, ctypes.byref(d), ctypes.byref(vid)))
        return vid.value

    @staticmethod
    def vae_out_shape(grid, temporal_up=(True, True, False), out_ch=3):
        F, Ht, Wt = grid
        t = F
        for u in temporal_up:
            if u:
                t = 1 + 2 * (t - 1)
        return (t, 16 * Ht, 16 * Wt, out_ch)

    def vae_decode(self, vae, latent, grid, rank=0, out=None, temporal_up=(True, True, False), out_ch=3):
        """latent: host fp32 [F*Ht*Wt, 64] (numpy) or a CUDA tensor; returns the video
        [T_out, 16 Ht, 16 Wt, out_ch] fp32 (numpy, or `out` if given: numpy or CUDA tensor)."""
        shape = self.vae_out_shape(grid, temporal_up, out_ch)
        flags = 0
        n = int(np.prod(grid)) * 64
        if isinstance(latent, np.ndarray):
            latent = np.ascontiguousarray(latent, dtype=np.float32)
            if latent.size != n:
                raise ValueError(f"latent has {latent.size} floats, grid {grid} needs {n}")
            lp = latent.ctypes.data_as(ctypes.c_void_p)
        else:
            if latent.numel() != n:
                raise ValueError(f"latent has {latent.numel()} floats, grid {grid} needs {n}")
            lp, flags = latent.data_ptr(), 1
        if out is None:
            out = np.empty(shape, dtype=np.float32)
        if isinstance(out, np.ndarray):
            if out.size != int(np.prod(shape)) or out.dtype != np.float32 or not out.flags.c_contiguous:
                raise ValueError(f"out must be a C-contiguous float32 array of shape {shape}")
            op = out.ctypes.data_as(ctypes.c_void_p)
        else:
            op, flags = out.data_ptr(), flags | 2
        self._ck(self._lib.gs_vae_decode(self._h, vae, rank, lp, *grid, op, flags))
        return out

    def vae_decode_request(self, vae, req, grid, temporal_up=(True, True, False), out_ch=3):
        out = np.empty(self.vae_out_shape(grid, temporal_up, out_ch), dtype=np.float32)
        self._ck(self._lib.gs_vae_decode_request(self._h, vae, req, out.ctypes.data_as(ctypes.c_void_p)))
        return out

    def debug_conv3d(self, x, w, bias, out, T, H, W, Cp, k, Coutp, resid=None, out_cs=None, mode=0,
                     out_real=0):
        kt, kh, kw = k
        self._ck(self._lib.gs_debug_conv3d(self._h, _ptr(x), _ptr(w), _ptr(bias), _ptr(resid), _ptr(out), T, H,
                                           W, Cp, kt, kh, kw, Coutp, Coutp if out_cs is None else out_cs,
                                           mode, out_real))

    # ---------------------------------------------------------------- measurement
    def profile(self, enable=True, reset=True):
        self._ck(self._lib.gs_profile(self._h, int(enable), int(reset)))

    def stats(self):
        import json
        buf = ctypes.create_string_buffer(1 << 16)
        self._ck(self._lib.gs_stats(self._h, buf, len(buf)))
        return json.loads(buf.value.decode())

    def stream_ptr(self, rank=None):
        s = ctypes.c_void_p()
        self._ck(self._lib.gs_stream(self._h, self.rank if rank is None else rank, ctypes.byref(s)))
        return s.value

    # ---------------------------------------------------------------- debug entry points
    def debug_gemm(self, epi, M, N, K, A, W, bias, out, gate_a=None, gate_b=None, gate_b_stride=0,
                   row_req=None, dsig=None):
        ds = _fl(list(dsig) + [0.0] * (8 - len(dsig))) if dsig is not None else None
        self._ck(self._lib.gs_debug_gemm(self._h, epi, M, N, K, _ptr(A), _ptr(W), _ptr(bias),
                                         _ptr(out), _ptr(gate_a), _ptr(gate_b), gate_b_stride,
                                         _ptr(row_req), ds))

    def debug_gemm_ssq(self, M, N, K, A, W, bias, out, ssq, ssq_cols):
        self._ck(self._lib.gs_debug_gemm_ssq(self._h, M, N, K, _ptr(A), _ptr(W), _ptr(bias), _ptr(out),
                                             _ptr(ssq), ssq_cols))

    def debug_attention(self, q, k, v, o, heads, d, seq_off, seq_len, q_rs=None, kv_rs=None,
                        o_rs=None):
        q_rs = heads * d if q_rs is None else q_rs
        kv_rs = heads * d if kv_rs is None else kv_rs
        o_rs = heads * d if o_rs is None else o_rs
        self._ck(self._lib.gs_debug_attention(self._h, _ptr(q), _ptr(k), _ptr(v), _ptr(o), heads,
                                              d, q_rs, kv_rs, o_rs, _ints(seq_off),
                                              _ints(seq_len), len(seq_len)))

    def debug_block(self, model, layer, x, grids, tok_lo, n_rows, t, prompts=None):
        """prompts (cross-attention models): uint16 bf16 bits [nreq, text_len, text_dim]."""
        x = np.ascontiguousarray(x, dtype=np.float32).copy()
        flat = [g for grid in grids for g in grid]
        pp = None
        if prompts is not None:
            prompts = np.ascontiguousarray(prompts, dtype=np.uint16)
            pp = prompts.ctypes.data_as(ctypes.c_void_p)
        self._ck(self._lib.gs_debug_block(self._h, model, layer, x.ctypes.data_as(_FP), len(n_rows),
                                          _ints(flat), _ints(tok_lo), _ints(n_rows), _fl(t), pp))
        return x

    def debug_attention_trace(self, cta=0):
        """clock64 stamps of attention CTA `cta` (0, or 1 = CTA 0's pair peer for d = 128) of the
        last launch (needs GS_ATTN_TRACE=1 at process start)."""
        buf = np.zeros(2 * 16 * 64, dtype=np.uint64)
        self._ck(self._lib.gs_debug_attention_trace(buf.ctypes.data_as(ctypes.c_void_p), buf.size))
        return buf.reshape(2, 16, 32, 2)[cta]

    def debug_attention_ctatime(self, n_ctas):
        """[n_ctas, 4] per-CTA (entry ns, first-S ns, exit ns, SM id) of the last attention launch
        (needs GS_ATTN_TRACE=1 at process start)."""
        buf = np.zeros(n_ctas * 4, dtype=np.uint64)
        self._ck(self._lib.gs_debug_attention_ctatime(buf.ctypes.data_as(ctypes.c_void_p), buf.size))
        return buf.reshape(n_ctas, 4)

    def debug_time_embed(self, model, t, dim):
        e0 = np.zeros((len(t), dim), np.float32)
        e = np.zeros((len(t), 6 * dim), np.float32)
        self._ck(self._lib.gs_debug_time_embed(self._h, model, len(t), _fl(t),
                                               e0.ctypes.data_as(_FP), e.ctypes.data_as(_FP)))
        return e0, e
