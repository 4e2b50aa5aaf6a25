"""Seeded Wishart input generator (support, untimed; no method arithmetic).

GPU build: ``libpolsar_gen.so`` (``polsar_gen_wishart``); host twin:
``libpolsar_gen_cpu.so`` -- same source (wishart_core.h), bit-identical
output.  See include/polsar_gen.h for the law and the layout.
"""
from __future__ import annotations

import ctypes

import numpy as np

from .. import _build

_P, _I64, _INT, _D, _U32, _U64 = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double,
                                  ctypes.c_uint32, ctypes.c_uint64)
_gpu = None
_cpu = None


def _load_gpu():
    global _gpu
    if _gpu is None:
        _gpu = ctypes.CDLL(_build.build_target("libpolsar_gen"))
        _gpu.polsar_gen_wishart.restype = _INT
        _gpu.polsar_gen_wishart.argtypes = [_P, _I64, _INT, _I64, _I64, _I64, _I64, _INT, _U64,
                                            _U32, _INT, _P, _I64, _D, _P]
    return _gpu


def _load_cpu():
    global _cpu
    if _cpu is None:
        _cpu = ctypes.CDLL(_build.build_target("libpolsar_gen_cpu"))
        _cpu.polsar_gen_wishart_cpu.restype = _INT
        _cpu.polsar_gen_wishart_cpu.argtypes = [_P, _I64, _INT, _I64, _I64, _I64, _I64, _INT, _U64,
                                                _U32, _INT, _P, _I64, _D]
        _cpu.polsar_gen_wishart_pixels_cpu.restype = _INT
        _cpu.polsar_gen_wishart_pixels_cpu.argtypes = [_P, _I64, _P, _I64, _INT, _I64, _I64, _INT,
                                                       _U64, _U32, _INT, _P, _I64, _D]
        _cpu.polsar_gen_cpu_log.restype = _D
        _cpu.polsar_gen_cpu_log.argtypes = [_D]
        _cpu.polsar_gen_cpu_exp2.restype = _D
        _cpu.polsar_gen_cpu_exp2.argtypes = [_D]
        _cpu.polsar_gen_cpu_cossin.restype = None
        _cpu.polsar_gen_cpu_cossin.argtypes = [_D, _P, _P]
    return _cpu


def _code(dtype) -> int:
    s = str(np.dtype(dtype)) if isinstance(dtype, type) else str(dtype)
    if s.endswith("float32"):
        return 0
    if s.endswith("float64"):
        return 1
    raise TypeError(f"unsupported dtype {dtype}")


def generate(cfg, row_begin=0, row_end=None, device="cuda", table=None, height=None, ld=None,
             stream=None, out=None):
    """Rows [row_begin, row_end) of cfg's image on the GPU -> torch (9, ld).

    ``height`` overrides cfg.height (e.g. weak-scaling images of N x 10000
    rows); ``table`` may be passed to avoid rebuilding it."""
    import torch

    H = cfg.height if height is None else height
    row_end = H if row_end is None else row_end
    n = (row_end - row_begin) * cfg.width
    tdt = torch.float32 if cfg.dtype == "float32" else torch.float64
    ld = n if ld is None else ld
    if out is None:
        out = torch.empty((9, ld), dtype=tdt, device=device)
    tab_np = cfg.table(H) if table is None else table
    tab = torch.as_tensor(np.ascontiguousarray(tab_np), dtype=torch.float64, device=device)
    s = torch.cuda.current_stream() if stream is None else stream
    rc = _load_gpu().polsar_gen_wishart(out.data_ptr(), out.stride(0), _code(tdt), row_begin,
                                        row_end, cfg.width, H, cfg.looks, cfg.seed, cfg.stream,
                                        cfg.mode, tab.data_ptr(), tab.shape[0],
                                        cfg.near_singular_frac, s.cuda_stream)
    if rc != 0:
        raise RuntimeError(f"polsar_gen_wishart failed rc={rc}")
    s.synchronize()  # keep `tab` alive until the kernel has read it
    return out


def generate_cpu(cfg, row_begin=0, row_end=None, table=None, height=None):
    """Host twin: rows [row_begin, row_end) -> numpy (9, n), bit-identical to
    :func:`generate`."""
    H = cfg.height if height is None else height
    row_end = H if row_end is None else row_end
    n = (row_end - row_begin) * cfg.width
    dt = np.float32 if cfg.dtype == "float32" else np.float64
    out = np.empty((9, n), dtype=dt)
    tab = np.ascontiguousarray(cfg.table(H) if table is None else table, dtype=np.float64)
    rc = _load_cpu().polsar_gen_wishart_cpu(out.ctypes.data, n, _code(dt), row_begin, row_end,
                                            cfg.width, H, cfg.looks, cfg.seed, cfg.stream, cfg.mode,
                                            tab.ctypes.data, tab.shape[0], cfg.near_singular_frac)
    if rc != 0:
        raise RuntimeError(f"polsar_gen_wishart_cpu failed rc={rc}")
    return out


def generate_pixels_cpu(cfg, pix, table=None, height=None):
    """Host twin for listed global pixel indices (y*width + x) -> numpy (9, m)."""
    H = cfg.height if height is None else height
    pix = np.ascontiguousarray(pix, dtype=np.int64)
    dt = np.float32 if cfg.dtype == "float32" else np.float64
    out = np.empty((9, pix.size), dtype=dt)
    tab = np.ascontiguousarray(cfg.table(H) if table is None else table, dtype=np.float64)
    rc = _load_cpu().polsar_gen_wishart_pixels_cpu(pix.ctypes.data, pix.size, out.ctypes.data,
                                                   pix.size, _code(dt), cfg.width, H, cfg.looks,
                                                   cfg.seed, cfg.stream, cfg.mode, tab.ctypes.data,
                                                   tab.shape[0], cfg.near_singular_frac)
    if rc != 0:
        raise RuntimeError(f"polsar_gen_wishart_pixels_cpu failed rc={rc}")
    return out


def cpu_log(x: float) -> float:
    return _load_cpu().polsar_gen_cpu_log(x)


def cpu_exp2(x: float) -> float:
    return _load_cpu().polsar_gen_cpu_exp2(x)


def cpu_cossin(u: float):
    c, s = ctypes.c_double(), ctypes.c_double()
    _load_cpu().polsar_gen_cpu_cossin(u, ctypes.byref(c), ctypes.byref(s))
    return c.value, s.value


def generate_bands(cfg, nbands, device="cuda", stream_stride=100):
    """Multi-frequency image: nbands independent
    Wishart images of cfg's law, band b drawn with stream id cfg.stream +
    b * stream_stride, stacked as 9 * nbands planes (block b at 9b..9b+8)."""
    import dataclasses

    import torch
    parts = []
    for b in range(nbands):
        cb = dataclasses.replace(cfg, stream=cfg.stream + b * stream_stride)
        parts.append(generate(cb, device=device))
    return torch.cat(parts, dim=0).contiguous()


def generate_bands_cpu(cfg, nbands, stream_stride=100):
    import dataclasses
    return np.concatenate([generate_cpu(dataclasses.replace(cfg, stream=cfg.stream + b * stream_stride))
                           for b in range(nbands)], axis=0)
