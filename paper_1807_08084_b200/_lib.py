"""ctypes loader for libpolsar.so (the C-ABI declared in include/polsar.h).

Marshalling only: no arithmetic of the method happens in Python.  There is no
CPU fallback -- if the library cannot be loaded, every entry point raises.
"""
from __future__ import annotations

import ctypes
import os
import threading

from . import _build

P = ctypes.c_void_p
I64 = ctypes.c_int64
INT = ctypes.c_int
D = ctypes.c_double
SZ = ctypes.c_size_t
U8P = ctypes.c_void_p
U64P = ctypes.c_void_p

# name -> (restype, argtypes), mirroring include/polsar.h
SIGNATURES = {
    "polsar_inv_det": (INT, [P, P, U8P, I64, I64, INT, P]),
    "polsar_inv_det_cholesky": (INT, [P, P, U8P, I64, I64, INT, P]),
    "polsar_inv_det_blocks": (INT, [P, P, U8P, I64, I64, INT, INT, P]),
    "polsar_window_workspace_bytes": (SZ, [I64, I64, INT, INT]),
    "polsar_window_workspace_bytes_for": (SZ, [INT, I64, I64, INT, INT]),
    "polsar_window_distance": (INT, [P, I64, I64, I64, I64, I64, INT, D, D, P, P, INT, P]),
    "polsar_window_kl": (INT, [P, I64, I64, I64, I64, I64, INT, D, D, P, P, INT, P]),
    "polsar_nlm_filter": (INT, [P, I64, I64, I64, I64, I64, INT, D, D, P, P, P, I64, INT, P]),
    "polsar_checksum": (INT, [P, I64, I64, INT, INT, I64, U8P, U64P, P]),
    "polsar_inv_det_host": (INT, [P, P, U8P, I64, I64, INT, INT, P, SZ, P, P, P]),
    "polsar_host_chunk_pixels": (I64, [SZ, INT]),
    "polsar_last_error": (ctypes.c_char_p, []),
    "polsar_version": (INT, []),
}

_lib = None
_lib_lock = threading.Lock()


class PolsarError(RuntimeError):
    pass


def lib() -> ctypes.CDLL:
    """Load (building in-tree first if the .so is missing or stale).  The
    handle is published only once every signature is declared, so threads
    calling in concurrently never see an unconfigured library."""
    global _lib
    if _lib is not None:
        return _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        path = _build.TARGETS["libpolsar"]["out"]
        override = os.environ.get("POLSAR_LIB_OVERRIDE")  # development A/B builds only
        if override:
            path = override
        try:
            if not override:
                _build.build_target("libpolsar")
        except Exception as e:  # toolchain missing: only an existing .so will do
            if not os.path.exists(path):
                raise PolsarError(f"libpolsar.so is not built and cannot be built: {e}") from e
        try:
            handle = ctypes.CDLL(path)
        except OSError as e:
            raise PolsarError(f"cannot load {path}: {e}") from e
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = lib().polsar_last_error().decode()
        raise PolsarError(f"{what} failed (rc={rc}): {msg}")
