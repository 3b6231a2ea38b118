"""Thin Python binding of the labuf C ABI (include/la.h) — argument
marshalling only.  Every step of the path runs in the CUDA kernels of
liblabuf.so; PyTorch only provides device memory and streams.  There is no
fallback: if the shared library is missing or fails to load, importing the
binding raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
# LABUF_LIB: an alternative build of the same library (A/B timing of two
# builds on one box, tools/ab.sh); the default is the in-tree build.
LIB_PATH = os.environ.get("LABUF_LIB", os.path.join(_PKG, "liblabuf.so"))

LA_OK, LA_ERR_INVALID, LA_ERR_UNSUPPORTED, LA_ERR_CAPACITY, LA_ERR_MODE, LA_ERR_CUDA, LA_ERR_NCCL = range(7)
LA_DT_F32, LA_DT_BF16, LA_DT_F16 = 0, 1, 2
LA_MODE_CHUNKWISE, LA_MODE_DIRECT = 0, 1
LA_VARIANT_GDN, LA_VARIANT_GATED, LA_VARIANT_VANILLA = 0, 1, 2
LA_FLUSH_FULL, LA_FLUSH_FORCE, LA_FLUSH_RAW = 0, 1, 2   # RAW is a flag OR-ed into FULL/FORCE (mode ii)
STATUS_BITS = {"bad_alpha": 0x1, "bad_beta": 0x2, "nonfinite": 0x4, "bad_nacc": 0x8}

_STATUS_NAMES = {0: "LA_OK", 1: "LA_ERR_INVALID", 2: "LA_ERR_UNSUPPORTED", 3: "LA_ERR_CAPACITY",
                 4: "LA_ERR_MODE", 5: "LA_ERR_CUDA", 6: "LA_ERR_NCCL"}

# The exported entry points of include/la.h, in declaration order.
EXPORTS = (
    "la_buf_query", "la_buf_create", "la_buf_destroy", "la_request_reset", "la_request_release",
    "la_decode_mixed", "la_pool_info", "la_decode_step",
    "la_flush", "la_verify_drafts", "la_commit_accepted", "la_verify_branches", "la_commit_branch",
    "la_commit_append", "la_state_fork",
    "la_direct_short", "la_prefill",
    "la_recurrent_step", "la_recurrent_verify", "la_recurrent_commit", "la_set_overlap", "la_set_prefill_chunk",
    "la_set_auto_flush",
    "la_state_get", "la_state_set", "la_slot_info", "la_device_status", "la_kernel_launches", "la_last_error",
    "la_tp_unique_id", "la_tp_init", "la_tp_allgather", "la_tp_destroy",
)


class LaError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class LaConfig(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "max_slots", "n_qk_heads", "n_v_heads", "d_k", "d_v", "chunk", "max_drafts",
        "short_cap", "in_dtype", "u_dtype", "keep_raw", "validate", "block_tokens", "n_blocks",
        "state_slots", "variant")]


class LaSizes(ctypes.Structure):
    _fields_ = [("state_bytes", ctypes.c_size_t), ("buffer_bytes", ctypes.c_size_t),
                ("meta_bytes", ctypes.c_size_t), ("align", ctypes.c_size_t),
                ("capacity", ctypes.c_int32), ("off_k", ctypes.c_size_t),
                ("off_u", ctypes.c_size_t), ("off_g", ctypes.c_size_t),
                ("off_v", ctypes.c_size_t), ("off_b", ctypes.c_size_t),
                ("record_bytes", ctypes.c_size_t), ("block_tokens", ctypes.c_int32),
                ("n_blocks", ctypes.c_int32), ("max_blocks", ctypes.c_int32), ("n_states", ctypes.c_int32),
                ("off_sidx", ctypes.c_size_t), ("off_btab", ctypes.c_size_t), ("off_wl", ctypes.c_size_t)]


_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load liblabuf.so (build it with paper_2605_19049_b200.build).  Raises
    if it is missing: there is no non-CUDA path."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} not found: run `python -m paper_2605_19049_b200.build` "
                           "(the CUDA library is required; there is no fallback)")
    if "LABUF_NCCL_LIB" not in os.environ:
        # the tensor-parallel helpers dlopen NCCL; point them at the wheel's copy
        try:
            import nvidia.nccl as _nccl
            cand = os.path.join(list(_nccl.__path__)[0], "lib", "libnccl.so.2")
            if os.path.exists(cand):
                os.environ["LABUF_NCCL_LIB"] = cand
        except Exception:
            pass
    lib = ctypes.CDLL(path)
    P, I32, VP = ctypes.POINTER, ctypes.c_int32, ctypes.c_void_p
    FP = P(ctypes.c_float)
    sigs = {
        "la_buf_query": [P(LaConfig), P(LaSizes)],
        "la_buf_create": [P(LaConfig), VP, VP, VP, I32, P(VP)],
        "la_buf_destroy": [VP],
        "la_request_reset": [VP, I32, I32, I32, I32, VP],
        "la_request_release": [VP, I32, I32, VP],
        "la_decode_mixed": [VP, I32, VP, VP, VP, VP, VP, VP, VP, VP],
        "la_pool_info": [VP, P(I32), P(I32), P(I32), P(I32), I32, P(I32), P(I32)],
        "la_decode_step": [VP, I32, I32, VP, VP, VP, VP, VP, VP, VP],
        "la_flush": [VP, I32, I32, I32, VP],
        "la_verify_drafts": [VP, I32, I32, I32, VP, VP, VP, VP, VP, VP, VP],
        "la_commit_accepted": [VP, I32, I32, VP, VP],
        "la_commit_append": [VP, I32, I32, VP, VP],
        "la_verify_branches": [VP, I32, I32, I32, I32, VP, VP, VP, VP, VP, VP, VP],
        "la_commit_branch": [VP, I32, I32, VP, VP, VP],
        "la_state_fork": [VP, I32, I32, I32, VP],
        "la_direct_short": [VP, I32, I32, I32, VP, VP, VP, VP, VP, VP, VP],
        "la_prefill": [VP, I32, I32, I32, VP, VP, VP, VP, VP, VP, VP],
        "la_recurrent_step": [VP, I32, I32, VP, VP, VP, VP, VP, VP, VP],
        "la_recurrent_verify": [VP, I32, I32, I32, VP, VP, VP, VP, VP, VP, VP, VP],
        "la_recurrent_commit": [VP, I32, I32, I32, VP, VP, VP],
        "la_set_overlap": [VP, I32],
        "la_set_prefill_chunk": [VP, I32],
        "la_set_auto_flush": [VP, I32],
        "la_state_get": [VP, I32, VP, VP],
        "la_state_set": [VP, I32, VP, VP],
        "la_slot_info": [VP, I32, P(I32), P(I32), P(I32), P(I32)],
        "la_device_status": [VP, VP, P(ctypes.c_uint32), VP, VP, VP],
        "la_tp_unique_id": [VP],
        "la_tp_init": [VP, I32, I32, I32, P(VP)],
        "la_tp_allgather": [VP, VP, VP, ctypes.c_size_t, VP],
        "la_tp_destroy": [VP],
    }
    for name, args in sigs.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    lib.la_kernel_launches.argtypes = [VP]
    lib.la_kernel_launches.restype = ctypes.c_int64
    lib.la_last_error.argtypes = []
    lib.la_last_error.restype = ctypes.c_char_p
    _lib = lib
    return lib


def _check(st: int):
    if st != LA_OK:
        raise LaError(st, load_library().la_last_error().decode())


def make_config(max_slots, n_qk_heads=16, n_v_heads=32, chunk=16, max_drafts=0, short_cap=0,
                in_dtype="bf16", u_dtype="f32", keep_raw=False, validate=False, d=128,
                block_tokens=0, n_blocks=0, state_slots=0, variant="gdn") -> LaConfig:
    """block_tokens > 0: paged record blocks from a pool of n_blocks;
    state_slots > 0: a pool of that many states, -1: none, 0: one per slot."""
    dt = {"f32": LA_DT_F32, "bf16": LA_DT_BF16, "f16": LA_DT_F16}
    var = {"gdn": LA_VARIANT_GDN, "gated": LA_VARIANT_GATED, "vanilla": LA_VARIANT_VANILLA}
    return LaConfig(max_slots, n_qk_heads, n_v_heads, d, d, chunk, max_drafts, short_cap,
                    dt[in_dtype], dt[u_dtype], int(keep_raw), int(validate), int(block_tokens),
                    int(n_blocks), int(state_slots), var[variant])


def query(cfg: LaConfig) -> LaSizes:
    s = LaSizes()
    _check(load_library().la_buf_query(ctypes.byref(cfg), ctypes.byref(s)))
    return s


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


_TORCH_IN = {LA_DT_F32: torch.float32, LA_DT_BF16: torch.bfloat16}


@dataclass
class SlotInfo:
    occ: int
    len: int
    mode: int
    pending: int


class LaBuf:
    """One GDN layer's state pool + KV buffers over torch-allocated device memory."""

    def __init__(self, cfg: LaConfig, device=None):
        self.lib = load_library()
        self.cfg = cfg
        idx = torch.cuda.current_device() if device is None else (torch.device(device).index or 0)
        self.device = torch.device("cuda", idx)
        self.sizes = query(cfg)
        al = self.sizes.align

        def alloc(nbytes):
            raw = torch.empty(nbytes + al, dtype=torch.uint8, device=self.device)
            off = (-raw.data_ptr()) % al
            return raw, raw[off:off + nbytes]

        self._raw_state, self._state = alloc(self.sizes.state_bytes)
        self._raw_buf, self._buffer = alloc(self.sizes.buffer_bytes)
        self._raw_meta, self._meta = alloc(self.sizes.meta_bytes)
        self._meta.zero_()
        h = ctypes.c_void_p()
        _check(self.lib.la_buf_create(ctypes.byref(cfg), _ptr(self._state), _ptr(self._buffer),
                                      _ptr(self._meta), self.device.index, ctypes.byref(h)))
        self.h = h
        self.in_torch = _TORCH_IN[cfg.in_dtype]

    # ------------------------------------------------------------ views
    @property
    def state(self) -> torch.Tensor:
        """fp32 [S][Hv][d_v][d_k] view of the state pool (device); S = max_slots
        (state r = slot r) unless the handle has a state pool."""
        c = self.cfg
        return self._state.view(torch.float32).view(self.sizes.n_states, c.n_v_heads, c.d_v, c.d_k)

    @property
    def capacity(self) -> int:
        return self.sizes.capacity

    def records(self):
        """Views of the buffered records (K, U, G): for tests and debugging."""
        c, s = self.cfg, self.sizes
        T, nb = s.block_tokens, s.n_blocks     # records per block, blocks (= slots when contiguous)
        udt = torch.float32 if c.u_dtype == LA_DT_F32 else torch.float16
        isz = 4 if c.in_dtype == LA_DT_F32 else 2
        usz = 4 if c.u_dtype == LA_DT_F32 else 2
        nK = nb * c.n_qk_heads * T * c.d_k
        nU = nb * c.n_v_heads * T * c.d_v
        K = self._buffer[s.off_k:s.off_k + nK * isz].view(self.in_torch).view(nb, c.n_qk_heads, T, c.d_k)
        # u records are tile-major: [blocks][Hv][d_v/32][bt][32]
        U = self._buffer[s.off_u:s.off_u + nU * usz].view(udt).view(nb, c.n_v_heads, c.d_v // 32, T, 32)
        G = self._buffer[s.off_g:s.off_g + nb * c.n_v_heads * T * 4].view(torch.float32).view(
            nb, c.n_v_heads, T)
        return K, U, G

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.la_buf_destroy(self.h)
                self.h = None
        except Exception:
            pass

    # ------------------------------------------------------------ checks
    def _chk(self, t, dtype, shape, name):
        if t is None:
            raise ValueError(f"{name} is required")
        if t.device != self.device or t.dtype != dtype or tuple(t.shape) != tuple(shape) or not t.is_contiguous():
            raise ValueError(f"{name}: expected contiguous {dtype} {tuple(shape)} on {self.device}, "
                             f"got {t.dtype} {tuple(t.shape)} on {t.device}")

    def _tok(self, n, n_tok, q, k, v, alpha, beta, o, o_required=True):
        c = self.cfg
        self._chk(q, self.in_torch, (n, n_tok, c.n_qk_heads, c.d_k), "q")
        self._chk(k, self.in_torch, (n, n_tok, c.n_qk_heads, c.d_k), "k")
        self._chk(v, self.in_torch, (n, n_tok, c.n_v_heads, c.d_v), "v")
        self._chk(alpha, torch.float32, (n, n_tok, c.n_v_heads), "alpha")
        self._chk(beta, torch.float32, (n, n_tok, c.n_v_heads), "beta")
        if o is not None or o_required:
            self._chk(o, torch.float32, (n, n_tok, c.n_v_heads, c.d_v), "o")

    # ------------------------------------------------------------ API
    def reset(self, first=0, n=None, mode=LA_MODE_CHUNKWISE, zero_state=True):
        n = self.cfg.max_slots - first if n is None else n
        _check(self.lib.la_request_reset(self.h, first, n, mode, int(zero_state), _stream()))

    def decode_step(self, first, q, k, v, alpha, beta, o):
        """q,k [n,Hk,d]; v [n,Hv,d]; alpha,beta [n,Hv]; o [n,Hv,d] (1 token per slot)."""
        n = q.shape[0]
        self._tok(n, 1, q.unsqueeze(1), k.unsqueeze(1), v.unsqueeze(1), alpha.unsqueeze(1),
                  beta.unsqueeze(1), o.unsqueeze(1))
        _check(self.lib.la_decode_step(self.h, first, n, _ptr(q), _ptr(k), _ptr(v), _ptr(alpha),
                                       _ptr(beta), _ptr(o), _stream()))

    def release(self, first=0, n=None):
        """Return slots' record blocks and states to the pools (la_request_release)."""
        n = self.cfg.max_slots - first if n is None else n
        _check(self.lib.la_request_release(self.h, first, n, _stream()))

    def decode_mixed(self, slots, q, k, v, alpha, beta, o):
        """One token per slot of an index-array batch in each slot's own form
        (la_decode_mixed).  slots: host int sequence (numpy / list); tensors
        q,k [n,Hk,d], v [n,Hv,d], alpha,beta [n,Hv], o [n,Hv,d] by batch row."""
        import numpy as np
        sl = slots if isinstance(slots, np.ndarray) and slots.dtype == np.int32 and slots.flags.c_contiguous \
            else np.ascontiguousarray(np.asarray(slots, dtype=np.int32))
        n = int(sl.shape[0])
        self._tok(n, 1, q.unsqueeze(1), k.unsqueeze(1), v.unsqueeze(1), alpha.unsqueeze(1),
                  beta.unsqueeze(1), o.unsqueeze(1))
        _check(self.lib.la_decode_mixed(self.h, n, sl.ctypes.data_as(ctypes.c_void_p), _ptr(q), _ptr(k),
                                        _ptr(v), _ptr(alpha), _ptr(beta), _ptr(o), _stream()))

    def pool_info(self, slot=-1):
        """dict: free/total blocks and states; with slot >= 0 also its block count and state index."""
        v = [ctypes.c_int32() for _ in range(6)]
        _check(self.lib.la_pool_info(self.h, *(ctypes.byref(x) for x in v[:4]), slot, ctypes.byref(v[4]),
                                     ctypes.byref(v[5])))
        out = {"free_blocks": v[0].value, "total_blocks": v[1].value, "free_states": v[2].value,
               "total_states": v[3].value}
        if slot >= 0:
            out["slot_blocks"], out["slot_state"] = v[4].value, v[5].value
        return out

    def flush(self, first=0, n=None, kind=LA_FLUSH_FULL):
        n = self.cfg.max_slots - first if n is None else n
        _check(self.lib.la_flush(self.h, first, n, kind, _stream()))

    def verify_drafts(self, first, q, k, v, alpha, beta, o):
        """Inputs [n, N, H, d] / [n, N, Hv]; o [n, N, Hv, d]."""
        n, N = q.shape[0], q.shape[1]
        self._tok(n, N, q, k, v, alpha, beta, o)
        _check(self.lib.la_verify_drafts(self.h, first, n, N, _ptr(q), _ptr(k), _ptr(v),
                                         _ptr(alpha), _ptr(beta), _ptr(o), _stream()))

    def commit_accepted(self, first, n_accepted):
        self._chk(n_accepted, torch.int32, (n_accepted.shape[0],), "n_accepted")
        _check(self.lib.la_commit_accepted(self.h, first, n_accepted.shape[0], _ptr(n_accepted),
                                           _stream()))

    def verify_branches(self, first, n_branch, q, k, v, alpha, beta, o):
        """n_branch candidate branches per slot, inputs [n, n_branch * n_draft, ...] branch-major."""
        n, tot = q.shape[0], q.shape[1]
        if tot % n_branch:
            raise ValueError("tokens per slot must be n_branch x n_draft")
        self._tok(n, tot, q, k, v, alpha, beta, o)
        _check(self.lib.la_verify_branches(self.h, first, n, n_branch, tot // n_branch, _ptr(q), _ptr(k), _ptr(v),
                                           _ptr(alpha), _ptr(beta), _ptr(o), _stream()))

    def commit_branch(self, first, branch, n_accepted):
        self._chk(branch, torch.int32, (branch.shape[0],), "branch")
        self._chk(n_accepted, torch.int32, (branch.shape[0],), "n_accepted")
        _check(self.lib.la_commit_branch(self.h, first, branch.shape[0], _ptr(branch), _ptr(n_accepted), _stream()))

    def commit_append(self, first, n_accepted):
        """Multi-round speculation: keep the accepted drafts buffered (la_commit_append)."""
        self._chk(n_accepted, torch.int32, (n_accepted.shape[0],), "n_accepted")
        _check(self.lib.la_commit_append(self.h, first, n_accepted.shape[0], _ptr(n_accepted), _stream()))

    def state_fork(self, src, dst, n_records):
        """dst's state <- src's state after its first n_records records (la_state_fork)."""
        _check(self.lib.la_state_fork(self.h, src, dst, n_records, _stream()))

    def direct_short(self, first, q, k, v, alpha, beta, o):
        n, m = q.shape[0], q.shape[1]
        self._tok(n, m, q, k, v, alpha, beta, o)
        _check(self.lib.la_direct_short(self.h, first, n, m, _ptr(q), _ptr(k), _ptr(v),
                                        _ptr(alpha), _ptr(beta), _ptr(o), _stream()))

    def prefill(self, first, q, k, v, alpha, beta, o=None):
        n, m = q.shape[0], q.shape[1]
        self._tok(n, m, q, k, v, alpha, beta, o, o_required=False)
        _check(self.lib.la_prefill(self.h, first, n, m, _ptr(q), _ptr(k), _ptr(v), _ptr(alpha),
                                   _ptr(beta), _ptr(o), _stream()))

    def recurrent_step(self, first, q, k, v, alpha, beta, o):
        n = q.shape[0]
        self._tok(n, 1, q.unsqueeze(1), k.unsqueeze(1), v.unsqueeze(1), alpha.unsqueeze(1),
                  beta.unsqueeze(1), o.unsqueeze(1))
        _check(self.lib.la_recurrent_step(self.h, first, n, _ptr(q), _ptr(k), _ptr(v),
                                          _ptr(alpha), _ptr(beta), _ptr(o), _stream()))

    def recurrent_verify(self, first, q, k, v, alpha, beta, temp, o):
        n, N = q.shape[0], q.shape[1]
        c = self.cfg
        self._tok(n, N, q, k, v, alpha, beta, o)
        self._chk(temp, torch.float32, (n, N, c.n_v_heads, c.d_v, c.d_k), "temp")
        _check(self.lib.la_recurrent_verify(self.h, first, n, N, _ptr(q), _ptr(k), _ptr(v),
                                            _ptr(alpha), _ptr(beta), _ptr(temp), _ptr(o), _stream()))

    def recurrent_commit(self, first, n_accepted, temp):
        n, N = temp.shape[0], temp.shape[1]
        self._chk(n_accepted, torch.int32, (n,), "n_accepted")
        _check(self.lib.la_recurrent_commit(self.h, first, n, N, _ptr(n_accepted), _ptr(temp),
                                            _stream()))

    def set_overlap(self, enable=True):
        """Programmatic dependent launch for this handle's kernels (la_set_overlap)."""
        _check(self.lib.la_set_overlap(self.h, 1 if enable else 0))

    def set_prefill_chunk(self, tokens=0):
        """Prefill chunk length (la_set_prefill_chunk; 0 = the handle's chunk)."""
        _check(self.lib.la_set_prefill_chunk(self.h, int(tokens)))

    def set_auto_flush(self, enable=True):
        """Fold a slot's buffer inside the decode step that fills it (la_set_auto_flush)."""
        _check(self.lib.la_set_auto_flush(self.h, 1 if enable else 0))

    def state_get(self, slot, dst=None):
        c = self.cfg
        if dst is None:
            dst = torch.empty(c.n_v_heads, c.d_v, c.d_k, dtype=torch.float32, device=self.device)
        self._chk(dst, torch.float32, (c.n_v_heads, c.d_v, c.d_k), "dst")
        _check(self.lib.la_state_get(self.h, slot, _ptr(dst), _stream()))
        return dst

    def state_set(self, slot, src):
        c = self.cfg
        self._chk(src, torch.float32, (c.n_v_heads, c.d_v, c.d_k), "src")
        _check(self.lib.la_state_set(self.h, slot, _ptr(src), _stream()))

    def slot_info(self, slot) -> SlotInfo:
        o, l, m, p = (ctypes.c_int32() for _ in range(4))
        _check(self.lib.la_slot_info(self.h, slot, ctypes.byref(o), ctypes.byref(l), ctypes.byref(m),
                                     ctypes.byref(p)))
        return SlotInfo(o.value, l.value, m.value, p.value)

    def device_status(self):
        """Synchronise; return (status flags, device occ, len, mode as int lists)."""
        R = self.cfg.max_slots
        f = ctypes.c_uint32()
        arrs = [(ctypes.c_int32 * R)() for _ in range(3)]
        _check(self.lib.la_device_status(self.h, _stream(), ctypes.byref(f),
                                         *[ctypes.cast(a, ctypes.c_void_p) for a in arrs]))
        return f.value, [list(a) for a in arrs]

    def kernel_launches(self) -> int:
        return int(self.lib.la_kernel_launches(self.h))


# ------------------------------------------------------------ tensor parallel
def tp_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load_library().la_tp_unique_id(buf))
    return buf.raw


class TPComm:
    """NCCL communicator for the tensor-parallel-over-heads configuration."""

    def __init__(self, unique_id: bytes, rank: int, world: int, device: int):
        self.lib = load_library()
        buf = ctypes.create_string_buffer(unique_id, 128)
        h = ctypes.c_void_p()
        _check(self.lib.la_tp_init(buf, rank, world, device, ctypes.byref(h)))
        self.h = h

    def allgather(self, send: torch.Tensor, recv: torch.Tensor):
        nb = send.numel() * send.element_size()
        if recv.numel() * recv.element_size() % nb:
            raise ValueError("recv size must be a multiple of send size")
        _check(self.lib.la_tp_allgather(self.h, _ptr(send), _ptr(recv), nb, _stream()))

    def destroy(self):
        if self.h:
            _check(self.lib.la_tp_destroy(self.h))
            self.h = None
