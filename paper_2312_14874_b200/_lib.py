"""ctypes binding of libprefixscan_b200.so (the C-ABI in include/prefixscan_b200.h).

There is no fallback: if the library is missing it is built with nvcc, and if
that is impossible every entry point raises.  The product path never touches
the CPU oracle.
"""

from __future__ import annotations

import ctypes
import os
import threading

from . import _build

PS_DTYPE = {"int32": 1, "int64": 2, "uint32": 3, "uint64": 4, "float32": 5, "float64": 6, "uint8": 7}
PS_ERR_DTYPE, PS_ERR_ARG, PS_ERR_SCRATCH, PS_ERR_EPOCH, PS_ERR_OVERLAP = 1, 2, 3, 4, 5
PS_ERR_CUDA_BASE = 1000
PS_EPOCH_MAX = 0x3FFFFFFF

_vp, _i64, _i32, _u32, _u64, _sz = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_uint32,
                                    ctypes.c_uint64, ctypes.c_size_t)

# name -> (restype, argtypes); must match include/prefixscan_b200.h exactly
SIGNATURES = {
    "ps_version": (_i32, []),
    "ps_pair_supported": (_i32, [_i32, _i32]),
    "ps_error_string": (ctypes.c_char_p, [_i32]),
    "ps_scan_scratch_bytes": (_sz, [_i64, _i32, _i32]),
    "ps_scan": (_i32, [_vp, _vp, _i64, _i32, _i32, _i32, _u64, _vp, _i64, _vp, _vp, _sz, _u32, _vp]),
    "ps_reduce_scratch_bytes": (_sz, [_i64, _i32]),
    "ps_reduce": (_i32, [_vp, _i64, _i32, _u64, _vp, _i64, _vp, _vp, _sz, _vp]),
    "ps_add_offset": (_i32, [_vp, _i64, _i32, _u64, _vp, _i64, _vp]),
    "ps_scan_batched_scratch_bytes": (_sz, [_i64, _i64, _i32, _i32]),
    "ps_scan_batched": (_i32, [_vp, _vp, _i64, _i64, _i64, _i64, _i32, _i32, _i32, _vp, _vp, _vp, _sz, _u32, _vp]),
    "ps_scan_segmented_scratch_bytes": (_sz, [_i64, _i32, _i32]),
    "ps_scan_segmented": (_i32, [_vp, _vp, _i64, _vp, _i64, _i32, _i32, _i32, _vp, _vp, _sz, _u32, _vp]),
    "ps_shift_right_scratch_bytes": (_sz, [_i64, _i32]),
    "ps_shift_right": (_i32, [_vp, _vp, _i64, _i32, _u64, _vp, _vp, _sz, _vp]),
    "ps_reduce_batched": (_i32, [_vp, _i64, _i64, _i64, _i32, _vp, _vp]),
    "ps_add_offset_batched": (_i32, [_vp, _i64, _i64, _i64, _i32, _vp, _vp]),
    "ps_reduce_wrapped_blocks": (_i32, [_vp, _i64, _i32, _u64, _vp, _vp]),
    "ps_scan_host_workspace_bytes": (_sz, [_i64, _i32, _i32]),
    "ps_scan_host_epochs": (_i64, [_i64, _i64]),
    "ps_set_tuning": (_i32, [ctypes.c_char_p, _i64]),
    "ps_get_tuning": (_i64, [ctypes.c_char_p]),
    "ps_scan_host": (_i32, [_vp, _vp, _i64, _i32, _i32, _i32, _u64, _vp, _vp, _sz, _i64, _u32, _vp]),
    "ps_scan_batched_host_workspace_bytes": (_sz, [_i64, _i64, _i32, _i32]),
    "ps_scan_batched_host": (_i32, [_vp, _vp, _i64, _i64, _i32, _i32, _i32, _vp, _sz, _i64, _u32, _vp]),
    "ps_host_register": (_i32, [_vp, _sz, ctypes.POINTER(_i32)]),
    "ps_host_unregister": (_i32, [_vp]),
    "ps_host_is_pinned": (_i32, [_vp]),
    "ps_tree_up_sweep": (_i32, [_vp, _i64, _i32, _vp, _vp]),
    "ps_tree_down_sweep": (_i32, [_vp, _i64, _i32, _vp]),
    "ps_publish_total": (_i32, [_vp, _vp, _i32, _i32, _u32, _u32, _vp, _vp, _vp]),
    "ps_scan_mailbox": (_i32, [_vp, _vp, _i64, _i32, _i32, _i32, _u64, _vp, _i32, _u32, _vp, _vp, _vp, _sz, _u32,
                               _vp]),
    "ps_select_scratch_bytes": (_sz, [_i64]),
    "ps_select": (_i32, [_vp, _vp, _i64, _i32, _i32, _i32, _vp, _vp, _vp, _sz, _u32, _vp]),
}

_lib = None
_lock = threading.Lock()


class ScanLibraryError(RuntimeError):
    """The native library is missing, failed to build, or a CUDA call failed."""


def load():
    """Load (building first if needed) the sm_100a library; raises if impossible."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            path = _build.LIB_PATH
            if not _build.up_to_date():
                try:
                    _build.build()
                except Exception as exc:  # no nvcc / compile error: no silent fallback
                    if not os.path.exists(path):
                        raise ScanLibraryError(f"cannot build {path}: {exc}") from exc
            try:
                lib = ctypes.CDLL(path)
            except OSError as exc:
                raise ScanLibraryError(f"cannot load {path}: {exc}") from exc
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def error_string(code: int) -> str:
    return load().ps_error_string(code).decode()


def check(code: int, what: str) -> None:
    """Map a C-ABI return code to the reference's exception classes:
    misuse -> ValueError (like core.py:69-78 / engine.py:94-105), CUDA or
    runtime failure -> RuntimeError (like engine.py:241-243)."""
    if code == 0:
        return
    msg = f"{what}: {error_string(code)} (code {code})"
    if code >= PS_ERR_CUDA_BASE:
        raise ScanLibraryError(msg)
    raise ValueError(msg)
