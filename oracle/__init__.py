"""ORACLE — TEST INFRASTRUCTURE ONLY.

Plain, slow fp64 CPU reference for the KV-buffered Gated DeltaNet decode path
of arxiv 2605.19049 ("the paper"; citations ``P:n`` = /root/reference/PAPER.md
line n).  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product (``paper_2605_19049_b200``) never imports, links or executes anything
here, and this package imports nothing from the product.

Contents
--------
``gdn_oracle.c`` / :func:`gdn_run`
    The plain definition: the GDN recurrence token by token,
    north-star convention S in R^{d_v x d_k} (reading Z1).  Every
    GPU output and every committed state is compared against this.
:mod:`oracle.forms`
    Independent fp64 implementations of the paper's *other* computation forms
    (chunkwise single-token P:403-407, chunkwise matrix form P:392-399,
    parallel form P:374-378, verify-then-commit P:173-177).  They are used
    only by the self-tests that prove the buffered forms equal the recurrence;
    the GPU path is never compared against them.

Pins: ``tests/test_oracle.py`` checks the recurrence against closed forms
(orthonormal keys, vanilla-LA brute force, beta = 0 decay, unit-key
overwrite, exact rational arithmetic on tiny inputs) and the forms against
the recurrence.  No function here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gdn_oracle.c")
_LIB_PATH = os.path.join(_HERE, "libgdn_oracle.so")
_lib = None
_lock = threading.Lock()


def build(force: bool = False) -> str:
    """Compile gdn_oracle.c with plain gcc -O2 (no SIMD intrinsics)."""
    if force or not os.path.exists(_LIB_PATH) or (
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC)):
        cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-o", _LIB_PATH,
               _SRC, "-lpthread"]
        subprocess.check_call(cmd)
    return _LIB_PATH


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB_PATH)
            dp = ctypes.POINTER(ctypes.c_double)
            lib.oracle_gdn_run.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_int, dp, dp, dp, dp, dp, dp, dp,
                                           dp, ctypes.c_int]
            lib.oracle_gdn_run.restype = ctypes.c_int
            _lib = lib
    return _lib


def _f64(a, shape):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if a.shape != tuple(shape):
        raise ValueError(f"expected shape {tuple(shape)}, got {a.shape}")
    return a


def _ptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def default_threads() -> int:
    return max(1, len(os.sched_getaffinity(0)))


def gdn_run(S, q, k, v, alpha, beta, beta_w=None, want_o=True, n_threads=None):
    """Advance independent GDN sequences token by token.

    S      [n_seq, d_v, d_k] start state (not modified; a copy is advanced)
    q, k   [n_seq, n_tok, d_k];  v [n_seq, n_tok, d_v]
    alpha, beta [n_seq, n_tok]; beta is the erase coefficient beta_e and,
    unless ``beta_w`` is given, also the write coefficient (GDN ties them).
    Returns (o [n_seq, n_tok, d_v] or None, S_end [n_seq, d_v, d_k]), fp64.
    Stored bf16/fp32 input values are widened to fp64 exactly.
    """
    S = np.array(S, dtype=np.float64, copy=True, order="C")
    n_seq, d_v, d_k = S.shape
    q = np.asarray(q)
    n_tok = q.shape[1]
    q = _f64(q, (n_seq, n_tok, d_k))
    k = _f64(k, (n_seq, n_tok, d_k))
    v = _f64(v, (n_seq, n_tok, d_v))
    alpha = _f64(alpha, (n_seq, n_tok))
    beta_e = _f64(beta, (n_seq, n_tok))
    beta_w = beta_e if beta_w is None else _f64(beta_w, (n_seq, n_tok))
    o = np.zeros((n_seq, n_tok, d_v), dtype=np.float64) if want_o else None
    lib = _load()
    rc = lib.oracle_gdn_run(n_seq, d_k, d_v, n_tok, _ptr(S), _ptr(q), _ptr(k), _ptr(v),
                            _ptr(alpha), _ptr(beta_e), _ptr(beta_w),
                            _ptr(o) if o is not None else None,
                            int(n_threads or default_threads()))
    if rc != 0:
        raise RuntimeError("oracle_gdn_run failed")
    return o, S
