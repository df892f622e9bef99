"""The C-ABI library loads on a CPU-only host and exports exactly what
include/prefixscan_b200.h declares; argument validation answers without a
GPU.  (No compute calls here -- those are the -m gpu tests.)"""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "prefixscan_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ps_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2312_14874_b200 import _lib
    return _lib.load()


def test_header_declares_the_hot_path_entry_points():
    names = declared_functions()
    for must in ("ps_scan", "ps_reduce", "ps_add_offset", "ps_scan_batched", "ps_scan_segmented",
                 "ps_shift_right", "ps_scan_host", "ps_error_string"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    for name in declared_functions():
        assert hasattr(lib, name), f"{name} declared in the header but not exported"


def test_python_binding_covers_every_declared_symbol():
    from paper_2312_14874_b200 import _lib
    assert set(_lib.SIGNATURES) == set(declared_functions())


def test_exports_are_plain_c_symbols():
    from paper_2312_14874_b200 import _build
    out = os.popen(f"nm -D --defined-only {_build.LIB_PATH}").read()
    exported = set(re.findall(r" T (ps_[a-z0-9_]+)$", out, flags=re.M))
    assert set(declared_functions()) <= exported


def test_library_is_sm100a():
    from paper_2312_14874_b200 import _build
    out = os.popen(f"cuobjdump --list-elf {_build.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out


def test_dtype_pairs(lib):
    codes = {"i32": 1, "i64": 2, "u32": 3, "u64": 4, "f32": 5, "f64": 6}
    ok = {("i32", "i32"), ("i32", "i64"), ("i64", "i64"), ("u32", "u32"), ("u32", "u64"), ("u64", "u64"),
          ("f32", "f32"), ("f32", "f64"), ("f64", "f64")}
    for a in codes:
        for b in codes:
            assert lib.ps_pair_supported(codes[a], codes[b]) == ((a, b) in ok), (a, b)


def test_validation_without_gpu(lib):
    from paper_2312_14874_b200 import _lib
    # bad dtype pair / negative n / bad epoch are rejected before any CUDA call
    assert lib.ps_scan(None, None, 10, 5, 2, 0, 0, None, 0, None, None, 0, 1, None) == _lib.PS_ERR_DTYPE
    assert lib.ps_scan(None, None, -1, 2, 2, 0, 0, None, 0, None, None, 0, 1, None) == _lib.PS_ERR_ARG
    assert lib.ps_scan(None, None, 4, 2, 2, 0, 0, None, 0, None, None, 0, 0, None) == _lib.PS_ERR_ARG
    buf = ctypes.create_string_buffer(64)
    assert lib.ps_scan(buf, buf, 4, 2, 2, 0, 0, None, 0, None, None, 0, 0, None) == _lib.PS_ERR_EPOCH
    assert lib.ps_scan_batched(buf, buf, 2, 4, 3, 4, 2, 2, 0, None, None, None, 0, 1, None) == _lib.PS_ERR_ARG
    assert lib.ps_reduce(buf, 4, 9, 0, None, 0, buf, buf, 1 << 20, None) == _lib.PS_ERR_DTYPE
    assert lib.ps_add_offset(buf, -3, 2, 0, None, 0, None) == _lib.PS_ERR_ARG
    assert _lib.error_string(_lib.PS_ERR_SCRATCH).startswith("scratch")


def test_error_mapping_matches_reference_exception_classes():
    from paper_2312_14874_b200 import _lib
    with pytest.raises(ValueError):
        _lib.check(_lib.PS_ERR_ARG, "x")
    with pytest.raises(RuntimeError):
        _lib.check(_lib.PS_ERR_CUDA_BASE + 2, "x")


def test_scratch_sizes_grow_with_n(lib):
    a = lib.ps_scan_scratch_bytes(1 << 20, 2, 2)
    b = lib.ps_scan_scratch_bytes(1 << 24, 2, 2)
    assert 0 < a < b
    # 20 bytes of descriptors per 4096-element tile: < 0.1 % of the 16 B/elem traffic
    assert b < (1 << 24) * 16 // 500
    assert lib.ps_scan_scratch_bytes(10, 5, 2) == 0  # unsupported pair


def test_select_validation_without_gpu(lib):
    from paper_2312_14874_b200 import _lib
    buf = ctypes.create_string_buffer(256)
    # unsupported value / flag dtypes, bad mode, negative n, missing buffers, short scratch
    assert lib.ps_select(buf, buf, 4, 7, 1, 0, buf, None, buf, 256, 1, None) == _lib.PS_ERR_DTYPE
    assert lib.ps_select(buf, buf, 4, 1, 9, 0, buf, None, buf, 256, 1, None) == _lib.PS_ERR_DTYPE
    assert lib.ps_select(buf, buf, 4, 1, 1, 2, buf, None, buf, 256, 1, None) == _lib.PS_ERR_ARG
    assert lib.ps_select(buf, buf, -1, 1, 1, 0, buf, None, buf, 256, 1, None) == _lib.PS_ERR_ARG
    assert lib.ps_select(buf, buf, 4, 1, 1, 0, buf, None, buf, 256, 0, None) == _lib.PS_ERR_EPOCH
    assert lib.ps_select(None, buf, 4, 1, 1, 0, buf, None, buf, 256, 1, None) == _lib.PS_ERR_ARG
    a = ctypes.create_string_buffer(1 << 16)
    b = ctypes.create_string_buffer(1 << 16)
    c = ctypes.create_string_buffer(1 << 16)
    assert lib.ps_select(a, b, 16, 1, 1, 0, a, None, c, 1 << 16, 1, None) == _lib.PS_ERR_OVERLAP
    assert lib.ps_select(a, b, 16, 1, 1, 0, c, None, a, 8, 1, None) == _lib.PS_ERR_SCRATCH
    # scratch: the larger of the tile counts (8 bytes per 8192 elements) and the
    # single-pass descriptors (16 bytes per 4096-element portion, + one round of slack)
    assert lib.ps_select_scratch_bytes(0) == 256 + 257 * 16
    big = lib.ps_select_scratch_bytes(1 << 28)
    assert big == 256 + ((1 << 28) // 4096 + 257) * 16
    assert lib.ps_select_scratch_bytes(-1) == 0


def test_mailbox_exchange_validation_without_gpu(lib):
    from paper_2312_14874_b200 import _lib
    buf = ctypes.create_string_buffer(256)
    # ps_publish_total: total, peer_mailboxes, n_peers, rank, epoch, prev_epoch, own_mailbox, timeout, stream
    assert lib.ps_publish_total(None, buf, 2, 0, 1, 0, buf, None, None) == _lib.PS_ERR_ARG
    assert lib.ps_publish_total(buf, buf, 0, 0, 1, 0, buf, None, None) == _lib.PS_ERR_ARG
    assert lib.ps_publish_total(buf, buf, 2, 2, 1, 0, buf, None, None) == _lib.PS_ERR_ARG   # rank out of range
    assert lib.ps_publish_total(buf, buf, 2, 1, 1, 1, buf, None, None) == _lib.PS_ERR_EPOCH  # prev == epoch
    assert lib.ps_publish_total(buf, buf, 2, 1, 0, 0, buf, None, None) == _lib.PS_ERR_EPOCH
    assert lib.ps_publish_total(buf, buf, 2, 1, 2, 1, None, None, None) == _lib.PS_ERR_ARG  # prev needs own mailbox
    # ps_scan_mailbox: in, out, n, din, dout, excl, seed, mailbox, n_wait, mail_epoch, timeout, total, scratch,
    #                  scratch_bytes, epoch, stream
    assert lib.ps_scan_mailbox(buf, buf, 4, 5, 2, 0, 0, buf, 1, 1, None, None, buf, 256, 1, None) == _lib.PS_ERR_DTYPE
    assert lib.ps_scan_mailbox(buf, buf, 4, 2, 2, 0, 0, None, 1, 1, None, None, buf, 256, 1, None) == _lib.PS_ERR_ARG
    assert lib.ps_scan_mailbox(buf, buf, 4, 2, 2, 0, 0, buf, 1, 0, None, None, buf, 256, 1, None) == _lib.PS_ERR_EPOCH
    assert lib.ps_scan_mailbox(buf, buf, -1, 2, 2, 0, 0, buf, 1, 1, None, None, buf, 256, 1, None) == _lib.PS_ERR_ARG


def test_tuning_knobs_roundtrip(lib):
    from paper_2312_14874_b200 import _lib
    for key, good, bad in ((b"scan_kernel", 3, 4), (b"rows_kernel", 2, 3), (b"select_kernel", 2, 3),
                           (b"stall_prob", 1024, 1025), (b"stream_inflight", 0, 9),
                           (b"rows_dynamic", 0, 2),
                           (b"rows_multi", 0, 2),
                           (b"tiles_row_lead", 0, 2),
                           (b"reduce_blocks", 0, 2),
                           (b"add_chunked", 0, 2)):
        prev = lib.ps_get_tuning(key)
        assert lib.ps_set_tuning(key, good) == 0 and lib.ps_get_tuning(key) == good
        assert lib.ps_set_tuning(key, bad) == _lib.PS_ERR_ARG and lib.ps_get_tuning(key) == good
        assert lib.ps_set_tuning(key, prev) == 0
    assert lib.ps_get_tuning(b"no_such_knob") == -1
    assert lib.ps_set_tuning(b"no_such_knob", 1) == _lib.PS_ERR_ARG
