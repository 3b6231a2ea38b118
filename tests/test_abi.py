"""C-ABI checks that need no GPU (driver runs these with -m "not gpu").

* liblabuf.so loads and exports every function include/la.h declares;
* la_buf_query sizing follows the documented layout (include/la.h "layout",
  DESIGN.md "Data layout in HBM");
* config validation and the all-or-nothing argument checks that the host
  library performs BEFORE touching the device (include/la.h "contract").
Handles here are created over fake (aligned, never dereferenced) device
addresses: la_buf_create does not access device memory, and every call
below fails its host-side checks before any CUDA call is made.
"""
from __future__ import annotations

import ctypes
import os
import re
import subprocess

import pytest

from paper_2605_19049_b200 import build as B
from paper_2605_19049_b200 import labuf as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "la.h")


@pytest.fixture(scope="module")
def lib():
    B.build()
    return L.load_library()


def declared_functions():
    src = open(HEADER).read()
    return re.findall(r"LA_API\s+[\w\s\*]+?\b(la_\w+)\s*\(", src)


def test_header_declares_the_north_star_calls():
    names = set(declared_functions())
    for n in ("la_buf_create", "la_decode_step", "la_flush", "la_verify_drafts",
              "la_commit_accepted", "la_direct_short"):
        assert n in names, n
    assert tuple(declared_functions()) == L.EXPORTS


def test_every_declared_symbol_is_exported(lib):
    out = subprocess.check_output(["nm", "-D", "--defined-only", B.LIB], text=True)
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    for name in declared_functions():
        assert name in exported, name
        assert getattr(lib, name) is not None
    # nothing but the C ABI leaks out (hidden visibility for internals)
    la_syms = {s for s in exported if s.startswith("la_")}
    assert la_syms == set(declared_functions())


def test_library_targets_sm100a_only():
    out = subprocess.check_output(["cuobjdump", "--list-elf", B.LIB], text=True)
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def _cfg(**kw):
    base = dict(max_slots=8, n_qk_heads=16, n_v_heads=32, chunk=16, max_drafts=4, short_cap=64)
    base.update(kw)
    return L.make_config(**base)


def test_query_sizes_match_layout(lib):
    s = L.query(_cfg())
    R, Hk, Hv, d = 8, 16, 32, 128
    T = (max(16 + 4, 64) + 3) & ~3
    assert s.capacity == T
    assert s.align == 1024
    assert s.state_bytes == R * Hv * d * d * 4
    assert s.off_k == 0
    assert s.off_u >= R * Hk * T * d * 2 and s.off_u % 1024 == 0
    assert s.off_g >= s.off_u + R * Hv * T * d * 4 and s.off_g % 1024 == 0
    assert s.buffer_bytes >= s.off_g + R * Hv * T * 4
    # record: k (QK heads, bf16) + u (V heads, fp32) + G (fp32), SURVEY Appendix B
    assert s.record_bytes == Hk * d * 2 + Hv * d * 4 + Hv * 4 == 20608
    s16 = L.query(_cfg(u_dtype="f16"))
    assert s16.record_bytes == 12416
    s32 = L.query(_cfg(in_dtype="f32"))
    assert s32.record_bytes == 24704
    sraw = L.query(_cfg(keep_raw=True))
    assert sraw.record_bytes == 20608 + Hv * d * 2 + Hv * 4
    assert sraw.off_b > sraw.off_v > sraw.off_g


@pytest.mark.parametrize("kw,status", [
    (dict(d=64), L.LA_ERR_UNSUPPORTED),
    (dict(n_qk_heads=3, n_v_heads=32), L.LA_ERR_UNSUPPORTED),
    (dict(n_qk_heads=4, n_v_heads=32), L.LA_ERR_UNSUPPORTED),     # g = 8
    (dict(chunk=0), L.LA_ERR_INVALID),
    (dict(chunk=65), L.LA_ERR_INVALID),
    (dict(max_drafts=17), L.LA_ERR_INVALID),
    (dict(short_cap=129), L.LA_ERR_INVALID),
    (dict(max_slots=0), L.LA_ERR_INVALID),
    (dict(in_dtype="f16"), L.LA_ERR_UNSUPPORTED),
    (dict(u_dtype="bf16"), L.LA_ERR_UNSUPPORTED),                 # reading Z11
    (dict(in_dtype="f32", u_dtype="f16"), L.LA_ERR_UNSUPPORTED),
])
def test_config_rejections(lib, kw, status):
    with pytest.raises(L.LaError) as e:
        L.query(_cfg(**kw))
    assert e.value.status == status
    assert lib.la_last_error().decode()


FAKE = 1 << 40          # 1024-aligned fake device address, never dereferenced


def _fake_handle(lib, cfg):
    h = ctypes.c_void_p()
    st = lib.la_buf_create(ctypes.byref(cfg), ctypes.c_void_p(FAKE), ctypes.c_void_p(FAKE * 2),
                           ctypes.c_void_p(FAKE * 3), 0, ctypes.byref(h))
    assert st == L.LA_OK
    return h


def test_create_rejects_misaligned_and_null(lib):
    cfg = _cfg()
    h = ctypes.c_void_p()
    assert lib.la_buf_create(ctypes.byref(cfg), ctypes.c_void_p(FAKE + 16), ctypes.c_void_p(FAKE),
                             ctypes.c_void_p(FAKE), 0, ctypes.byref(h)) == L.LA_ERR_INVALID
    assert lib.la_buf_create(ctypes.byref(cfg), None, ctypes.c_void_p(FAKE),
                             ctypes.c_void_p(FAKE), 0, ctypes.byref(h)) == L.LA_ERR_INVALID
    assert lib.la_buf_create(ctypes.byref(cfg), ctypes.c_void_p(FAKE), ctypes.c_void_p(FAKE),
                             ctypes.c_void_p(FAKE), -1, ctypes.byref(h)) == L.LA_ERR_INVALID


def test_host_checks_before_any_device_work(lib):
    """Every rejection below happens before a CUDA call and leaves the host
    mirror unchanged (all-or-nothing)."""
    cfg = _cfg()
    h = _fake_handle(lib, cfg)
    P = ctypes.c_void_p
    ok = P(FAKE * 5)
    args = (ok, ok, ok, ok, ok, ok, None)
    # slot range outside [0, R)
    assert lib.la_decode_step(h, 4, 5, *args) == L.LA_ERR_INVALID
    assert lib.la_decode_step(h, -1, 1, *args) == L.LA_ERR_INVALID
    # null / misaligned inputs
    assert lib.la_decode_step(h, 0, 1, None, ok, ok, ok, ok, ok, None) == L.LA_ERR_INVALID
    assert lib.la_decode_step(h, 0, 1, P(FAKE + 2), ok, ok, ok, ok, ok, None) == L.LA_ERR_INVALID
    # n_draft outside [1, max_drafts]
    assert lib.la_verify_drafts(h, 0, 1, 0, *args) == L.LA_ERR_INVALID
    assert lib.la_verify_drafts(h, 0, 1, 5, *args) == L.LA_ERR_INVALID
    # direct on a CHUNKWISE slot; commit without a pending verify
    assert lib.la_direct_short(h, 0, 1, 1, *args) == L.LA_ERR_MODE
    assert lib.la_commit_accepted(h, 0, 1, ok, None) == L.LA_ERR_MODE
    assert lib.la_flush(h, 0, 1, 7, None) == L.LA_ERR_INVALID
    # an empty flush / empty range is a no-op, not an error
    assert lib.la_flush(h, 0, 8, L.LA_FLUSH_FULL, None) == L.LA_OK
    assert lib.la_decode_step(h, 0, 0, *args) == L.LA_OK
    # mirror unchanged
    o, ln, m, p = (ctypes.c_int32() for _ in range(4))
    for r in range(8):
        assert lib.la_slot_info(h, r, ctypes.byref(o), ctypes.byref(ln), ctypes.byref(m),
                                ctypes.byref(p)) == L.LA_OK
        assert (o.value, ln.value, m.value, p.value) == (0, 0, 0, 0)
    assert lib.la_kernel_launches(h) == 0
    assert lib.la_buf_destroy(h) == L.LA_OK


def test_direct_mode_disabled_without_short_cap(lib):
    h = _fake_handle(lib, _cfg(short_cap=0))
    assert lib.la_request_reset(h, 0, 1, L.LA_MODE_DIRECT, 0, None) == L.LA_ERR_MODE
    lib.la_buf_destroy(h)


def test_binding_has_no_fallback(tmp_path):
    """The binding refuses to run without the CUDA library (no CPU path)."""
    import importlib
    mod = importlib.import_module("paper_2605_19049_b200.labuf")
    saved = mod._lib
    try:
        mod._lib = None
        with pytest.raises(RuntimeError, match="no fallback"):
            mod.load_library(str(tmp_path / "missing.so"))
    finally:
        mod._lib = saved


def test_launch_options_and_raw_flag_validation(lib):
    """la_set_overlap / la_set_auto_flush accept 0/1 only; LA_FLUSH_RAW needs
    a keep_raw handle (rejected before any device work, mirror unchanged);
    the header and the binding agree on the flag values."""
    hdr = open(HEADER).read()
    assert "LA_FLUSH_RAW = 2" in hdr and L.LA_FLUSH_RAW == 2
    h = _fake_handle(lib, _cfg())
    for fn in (lib.la_set_overlap, lib.la_set_auto_flush):
        assert fn(h, 1) == L.LA_OK and fn(h, 0) == L.LA_OK
        assert fn(h, 2) == L.LA_ERR_INVALID and fn(h, -1) == L.LA_ERR_INVALID
        assert fn(None, 1) == L.LA_ERR_INVALID
    assert lib.la_flush(h, 0, 1, L.LA_FLUSH_FORCE | L.LA_FLUSH_RAW, None) == L.LA_ERR_INVALID
    assert lib.la_flush(h, 0, 1, L.LA_FLUSH_FULL | L.LA_FLUSH_RAW, None) == L.LA_ERR_INVALID
    assert lib.la_flush(h, 0, 1, 4 | L.LA_FLUSH_FULL, None) == L.LA_ERR_INVALID
    assert lib.la_kernel_launches(h) == 0
    lib.la_buf_destroy(h)
    # with keep_raw the raw flag passes the host checks (empty flush: no-op)
    h = _fake_handle(lib, _cfg(keep_raw=True))
    assert lib.la_flush(h, 0, 8, L.LA_FLUSH_FULL | L.LA_FLUSH_RAW, None) == L.LA_OK
    assert lib.la_kernel_launches(h) == 0
    lib.la_buf_destroy(h)


# ------------------------------------------------------------------ pools
def test_paged_sizes_and_state_pool(lib):
    """Paged handles size the buffer by the block pool (n_blocks x block_tokens
    records), a state pool sizes the state by state_slots, and meta
    carries the state index, block table and work lists (include/la.h)."""
    R, Hk, Hv, d = 8, 16, 32, 128
    s = L.query(_cfg(block_tokens=8, n_blocks=40, state_slots=5))
    T = 64
    assert (s.block_tokens, s.n_blocks, s.max_blocks, s.n_states) == (8, 40, T // 8, 5)
    assert s.state_bytes == 5 * Hv * d * d * 4
    assert s.off_u >= 40 * Hk * 8 * d * 2 and s.off_g >= s.off_u + 40 * Hv * 8 * d * 4
    assert s.buffer_bytes >= s.off_g + 40 * Hv * 8 * 4
    assert s.off_sidx == 4 * R * 4 + 16 and s.off_btab == s.off_sidx + R * 4
    assert s.off_wl == s.off_btab + R * (T // 8) * 4 and s.meta_bytes >= s.off_wl + 6 * R * 4
    c = L.query(_cfg())            # contiguous: one block of T records per slot, one state per slot
    assert (c.block_tokens, c.n_blocks, c.max_blocks, c.n_states) == (T, R, 1, R)
    assert L.query(_cfg(state_slots=-1)).state_bytes == 0     # KV-only handle


@pytest.mark.parametrize("kw", [dict(block_tokens=6, n_blocks=4), dict(block_tokens=8, n_blocks=0),
                                dict(block_tokens=132, n_blocks=4), dict(state_slots=-2)])
def test_pool_config_rejections(lib, kw):
    with pytest.raises(L.LaError) as e:
        L.query(_cfg(**kw))
    assert e.value.status == L.LA_ERR_INVALID


def test_state_pool_exhaustion_before_device_work(lib):
    """Without states (state_slots = -1) a slot cannot become CHUNKWISE, and a
    slot that holds no state cannot decode: both rejected on the host, before
    any CUDA call, pools and mirror unchanged."""
    h = _fake_handle(lib, _cfg(block_tokens=8, n_blocks=16, state_slots=-1))
    assert lib.la_request_reset(h, 0, 1, L.LA_MODE_CHUNKWISE, 0, None) == L.LA_ERR_CAPACITY
    P = ctypes.c_void_p
    ok = P(FAKE * 5)
    assert lib.la_decode_step(h, 0, 1, ok, ok, ok, ok, ok, ok, None) == L.LA_ERR_MODE
    sl = (ctypes.c_int32 * 2)(0, 0)
    assert lib.la_decode_mixed(h, 2, sl, ok, ok, ok, ok, ok, ok, None) == L.LA_ERR_MODE      # no state
    v = [ctypes.c_int32() for _ in range(6)]
    assert lib.la_pool_info(h, *(ctypes.byref(x) for x in v[:4]), 0, ctypes.byref(v[4]), ctypes.byref(v[5])) == L.LA_OK
    assert [x.value for x in v] == [16, 16, 0, 0, 0, -1]
    assert lib.la_kernel_launches(h) == 0
    lib.la_buf_destroy(h)
    h = _fake_handle(lib, _cfg())      # contiguous: every slot owns its state
    assert lib.la_decode_mixed(h, 2, sl, ok, ok, ok, ok, ok, ok, None) == L.LA_ERR_INVALID   # duplicate slot
    sl[1] = 8
    assert lib.la_decode_mixed(h, 2, sl, ok, ok, ok, ok, ok, ok, None) == L.LA_ERR_INVALID   # out of range
    assert lib.la_kernel_launches(h) == 0
    lib.la_buf_destroy(h)


def test_variant_field(lib):
    """la_config.variant: GDN / gated / vanilla accepted, anything else
    LA_ERR_INVALID; mode ii (LA_FLUSH_RAW) is the GDN UT transform only."""
    for v in ("gdn", "gated", "vanilla"):
        L.query(_cfg(variant=v))
    cfg = _cfg()
    cfg.variant = 3
    with pytest.raises(L.LaError) as e:
        L.query(cfg)
    assert e.value.status == L.LA_ERR_INVALID
    h = _fake_handle(lib, _cfg(keep_raw=True, variant="vanilla"))
    assert lib.la_flush(h, 0, 1, L.LA_FLUSH_FULL | L.LA_FLUSH_RAW, None) == L.LA_ERR_UNSUPPORTED
    lib.la_buf_destroy(h)
