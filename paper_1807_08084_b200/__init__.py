"""B200-native batched inverse + determinant of 3x3 Hermitian PD PolSAR
matrices (arXiv 1807.08084).

Thin Python binding over the C-ABI in ``include/polsar.h`` (same names; torch
is used only for device memory and streams).  Every step of the hot path runs
in the CUDA kernels of ``libpolsar.so``; there is no CPU fallback and the
oracle (``oracle/``) is never imported from here.

Tensors: ``z`` is (9, ld) -- the packed upper triangle a, Re b, Im b, Re c,
Im c, d, Re e, Im e, f as planes -- and ``out`` is (11, ld):
the inverse's 9 planes, det Z, det Z^-1.  float32 tensors select POLSAR_F32
(fp64 arithmetic) unless ``plain=True``; float64 tensors select POLSAR_F64
(Alg. 2 with ~2u cofactors and a compensated determinant) unless
``plain=True`` (Alg. 2 as printed) or ``eft=True`` (POLSAR_F64_EFT, the
error-free-transformation Alg. 2; inverse/det entry points only).
"""
from __future__ import annotations

import ctypes

from ._lib import PolsarError, check, lib

POLSAR_F32, POLSAR_F64, POLSAR_F32_PLAIN, POLSAR_F64_PLAIN, POLSAR_F64_EFT = 0, 1, 2, 3, 4
STATUS_OK, STATUS_SINGULAR, STATUS_NOT_PD = 0, 1, 2

__all__ = [
    "polsar_inv_det", "polsar_inv_det_cholesky", "polsar_inv_det_blocks", "polsar_window_distance",
    "polsar_nlm_filter", "nlm_filter", "polsar_window_kl", "window_kl", "polsar_window_workspace_bytes", "polsar_window_workspace_bytes_for", "polsar_checksum", "polsar_inv_det_host",
    "polsar_host_chunk_pixels", "inv_det", "window_distance", "dtype_code", "PolsarError",
    "POLSAR_F32", "POLSAR_F64", "POLSAR_F32_PLAIN", "POLSAR_F64_PLAIN", "POLSAR_F64_EFT",
]


def _torch():
    import torch
    return torch


def dtype_code(tdtype, plain: bool = False, eft: bool = False) -> int:
    torch = _torch()
    if plain and eft:
        raise ValueError("plain and eft are exclusive")
    if tdtype == torch.float32:
        if eft:
            raise ValueError("eft (POLSAR_F64_EFT) needs float64 storage")
        return POLSAR_F32_PLAIN if plain else POLSAR_F32
    if tdtype == torch.float64:
        return POLSAR_F64_PLAIN if plain else (POLSAR_F64_EFT if eft else POLSAR_F64)
    raise TypeError(f"unsupported dtype {tdtype}")


def _stream_ptr(stream):
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _dev_check(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise PolsarError("polsar kernels take CUDA tensors (no CPU fallback)")


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _planes(z, nplanes):
    if z.dim() != 2 or z.shape[0] != nplanes:
        raise ValueError(f"expected a ({nplanes}, ld) tensor, got {tuple(z.shape)}")
    if z.stride(1) != 1:
        raise ValueError("planes must be contiguous along pixels")
    return z.stride(0)


def _count(n, *tensors):
    """Pixel count: all of z's columns by default; an explicit n must fit in
    every tensor's pixel extent (a strided view's planes end at shape[1])."""
    lim = min(t.shape[1] for t in tensors)
    n = lim if n is None else int(n)
    if n < 0 or n > lim:
        raise ValueError(f"n = {n} outside [0, {lim}] (the tensors' pixel extent)")
    return n


def _inv_det_call(name, z, out, status, n, plain, stream, eft=False):
    _dev_check(z, out, status)
    ldz = _planes(z, 9)
    ldo = _planes(out, 11)
    if ldz != ldo:
        raise ValueError("z and out must share the plane stride ld")
    if out.dtype != z.dtype:
        raise TypeError("z and out must have the same dtype")
    n = _count(n, z, out)
    if status is not None and (status.dtype != _torch().uint8 or status.numel() < n):
        raise ValueError("status must be a uint8 tensor of >= n elements")
    rc = getattr(lib(), name)(_ptr(z), _ptr(out), _ptr(status), n, ldz,
                              dtype_code(z.dtype, plain, eft), _stream_ptr(stream))
    check(rc, name)
    return out


def polsar_inv_det(z, out, status=None, n=None, plain=False, stream=None, eft=False):
    """Alg. 2 on every pixel: out = [Z^-1 (9), det, 1/det]."""
    return _inv_det_call("polsar_inv_det", z, out, status, n, plain, stream, eft)


def polsar_inv_det_cholesky(z, out, status=None, n=None, plain=False, stream=None):
    """Alg. 1 (PAPER.md:279-378, l21 corrected) on every pixel."""
    return _inv_det_call("polsar_inv_det_cholesky", z, out, status, n, plain, stream)


def polsar_inv_det_blocks(z, out, nblocks, status=None, n=None, plain=False, stream=None, eft=False):
    """Multi-frequency block-diagonal pixels: z is
    (9*nblocks, ld), out (9*nblocks + 2, ld)."""
    _dev_check(z, out, status)
    ldz = _planes(z, 9 * nblocks)
    if _planes(out, 9 * nblocks + 2) != ldz:
        raise ValueError("z and out must share the plane stride ld")
    if out.dtype != z.dtype:
        raise TypeError("z and out must have the same dtype")
    n = _count(n, z, out)
    if status is not None and (status.dtype != _torch().uint8 or status.numel() < n):
        raise ValueError("status must be a uint8 tensor of >= n elements")
    rc = lib().polsar_inv_det_blocks(_ptr(z), _ptr(out), _ptr(status), n, ldz, int(nblocks),
                                     dtype_code(z.dtype, plain, eft), _stream_ptr(stream))
    check(rc, "polsar_inv_det_blocks")
    return out


def inv_det(z, algo: str = "adjugate", plain: bool = False, with_status: bool = True,
            stream=None, eft: bool = False):
    """Allocate outputs and run K1 (algo='adjugate') or K2 (algo='cholesky')."""
    torch = _torch()
    out = torch.empty((11, z.shape[1]), dtype=z.dtype, device=z.device)
    status = torch.empty(z.shape[1], dtype=torch.uint8, device=z.device) if with_status else None
    if algo == "adjugate":
        polsar_inv_det(z, out, status, plain=plain, stream=stream, eft=eft)
    else:
        if eft:
            raise ValueError("eft (POLSAR_F64_EFT) is an Alg. 2 mode")
        polsar_inv_det_cholesky(z, out, status, plain=plain, stream=stream)
    return (out, status) if with_status else out


def polsar_window_workspace_bytes(slab_rows: int, width: int, radius: int, dtype: int) -> int:
    return int(lib().polsar_window_workspace_bytes(slab_rows, width, radius, dtype))


WINDOW, NLM, KL = 0, 1, 2  # entry points of polsar_window_workspace_bytes_for


def polsar_window_workspace_bytes_for(entry: int, slab_rows: int, width: int, radius: int, dtype: int) -> int:
    return int(lib().polsar_window_workspace_bytes_for(int(entry), slab_rows, width, radius, dtype))


def polsar_window_distance(z, width, slab_rows, out_row_begin, out_row_end, radius, looks, h,
                           workspace, out, plain=False, stream=None):
    """Search-window sum W_i (BASELINE configs[4]) for slab rows
    [out_row_begin, out_row_end); out has (end - begin) * width elements."""
    _dev_check(z, workspace, out)
    ld = _planes(z, 9)
    code = dtype_code(z.dtype, plain)
    need = polsar_window_workspace_bytes_for(WINDOW, slab_rows, width, radius, code)
    if workspace.numel() * workspace.element_size() < need:
        raise ValueError(f"workspace needs {need} bytes")
    if out.numel() < (out_row_end - out_row_begin) * width or out.dtype != z.dtype:
        raise ValueError("out too small or wrong dtype")
    rc = lib().polsar_window_distance(_ptr(z), ld, width, slab_rows, out_row_begin, out_row_end,
                                      radius, float(looks), float(h), _ptr(workspace), _ptr(out),
                                      code, _stream_ptr(stream))
    check(rc, "polsar_window_distance")
    return out


def window_distance(z, height, width, radius=11, looks=4.0, h=1.0, row_begin=0, row_end=None,
                    plain=False, stream=None):
    """Allocate and run K3 on a whole slab z of height x width pixels."""
    torch = _torch()
    row_end = height if row_end is None else row_end
    code = dtype_code(z.dtype, plain)
    ws = torch.empty(polsar_window_workspace_bytes_for(WINDOW, height, width, radius, code),
                     dtype=torch.uint8, device=z.device)
    out = torch.empty((row_end - row_begin) * width, dtype=z.dtype, device=z.device)
    return polsar_window_distance(z, width, height, row_begin, row_end, radius, looks, h, ws, out,
                                  plain=plain, stream=stream)


def polsar_window_kl(z, width, slab_rows, out_row_begin, out_row_end, radius, looks, h,
                     workspace, out, stream=None):
    """Window sum with the symmetric Wishart KL distance."""
    _dev_check(z, workspace, out)
    ld = _planes(z, 9)
    code = dtype_code(z.dtype)
    need = polsar_window_workspace_bytes_for(KL, slab_rows, width, radius, code)
    if workspace.numel() * workspace.element_size() < need:
        raise ValueError(f"workspace needs {need} bytes")
    if out.numel() < (out_row_end - out_row_begin) * width or out.dtype != z.dtype:
        raise ValueError("out too small or wrong dtype")
    rc = lib().polsar_window_kl(_ptr(z), ld, width, slab_rows, out_row_begin, out_row_end, radius,
                                float(looks), float(h), _ptr(workspace), _ptr(out), code,
                                _stream_ptr(stream))
    check(rc, "polsar_window_kl")
    return out


def window_kl(z, height, width, radius=11, looks=4.0, h=1.0, row_begin=0, row_end=None,
              stream=None):
    torch = _torch()
    row_end = height if row_end is None else row_end
    code = dtype_code(z.dtype)
    ws = torch.empty(max(1, polsar_window_workspace_bytes_for(KL, height, width, radius, code)),
                     dtype=torch.uint8, device=z.device)
    out = torch.empty((row_end - row_begin) * width, dtype=z.dtype, device=z.device)
    return polsar_window_kl(z, width, height, row_begin, row_end, radius, looks, h, ws, out,
                            stream=stream)


def polsar_nlm_filter(z, width, slab_rows, out_row_begin, out_row_end, radius, looks, h,
                      workspace, out_z, out_w=None, plain=False, stream=None):
    """NLM filter output Zhat (9 planes) and optionally W for slab rows
    [out_row_begin, out_row_end), with the K3 weights."""
    _dev_check(z, workspace, out_z, out_w)
    ld = _planes(z, 9)
    ld_out = _planes(out_z, 9)
    code = dtype_code(z.dtype, plain)
    need = polsar_window_workspace_bytes_for(NLM, slab_rows, width, radius, code)
    if workspace.numel() * workspace.element_size() < need:
        raise ValueError(f"workspace needs {need} bytes")
    if out_z.dtype != z.dtype or (out_w is not None and out_w.dtype != z.dtype):
        raise TypeError("outputs must have the input dtype")
    m = (out_row_end - out_row_begin) * width
    if out_z.shape[1] < m or (out_w is not None and out_w.numel() < m):
        raise ValueError(f"out_z / out_w must hold {m} pixels")
    if z.shape[1] < slab_rows * width:
        raise ValueError("z holds fewer than slab_rows * width pixels")
    rc = lib().polsar_nlm_filter(_ptr(z), ld, width, slab_rows, out_row_begin, out_row_end, radius,
                                 float(looks), float(h), _ptr(workspace), _ptr(out_w), _ptr(out_z),
                                 ld_out, code, _stream_ptr(stream))
    check(rc, "polsar_nlm_filter")
    return out_z


def nlm_filter(z, height, width, radius=11, looks=4.0, h=1.0, row_begin=0, row_end=None,
               plain=False, stream=None):
    """Allocate and run the fused NLM filter on a whole slab; returns (Zhat, W)."""
    torch = _torch()
    row_end = height if row_end is None else row_end
    m = (row_end - row_begin) * width
    code = dtype_code(z.dtype, plain)
    ws = torch.empty(polsar_window_workspace_bytes_for(NLM, height, width, radius, code),
                     dtype=torch.uint8, device=z.device)
    out_z = torch.empty((9, m), dtype=z.dtype, device=z.device)
    out_w = torch.empty(m, dtype=z.dtype, device=z.device)
    polsar_nlm_filter(z, width, height, row_begin, row_end, radius, looks, h, ws, out_z, out_w,
                      plain=plain, stream=stream)
    return out_z, out_w


def polsar_checksum(planes, n, nplanes, pix_offset=0, status=None, result=None, stream=None):
    """Order-independent hash of nplanes planes (+ status counts) -> result
    (device uint64[4], accumulated in place)."""
    torch = _torch()
    _dev_check(planes, status)
    if result is None:
        result = torch.zeros(4, dtype=torch.int64, device=planes.device)
    ld = planes.stride(0) if planes.dim() == 2 else planes.numel()
    code = POLSAR_F32 if planes.element_size() == 4 else POLSAR_F64
    rc = lib().polsar_checksum(_ptr(planes), n, ld, nplanes, code, pix_offset, _ptr(status),
                               _ptr(result), _stream_ptr(stream))
    check(rc, "polsar_checksum")
    return result


def polsar_host_chunk_pixels(ws_bytes: int, dtype: int) -> int:
    return int(lib().polsar_host_chunk_pixels(ws_bytes, dtype))


def polsar_inv_det_host(z_host, out_host, status_host, workspace, streams, algo=0, plain=False, eft=False):
    """End-to-end call on HOST tensors (pinned): chunked H2D / kernel / D2H
    pipeline over three CUDA streams; returns after the last copy."""
    if z_host.is_cuda or out_host.is_cuda:
        raise PolsarError("polsar_inv_det_host takes host tensors")
    ld = _planes(z_host, 9)
    if _planes(out_host, 11) != ld:
        raise ValueError("z_host and out_host must share the plane stride")
    n = _count(None, z_host, out_host)
    if status_host is not None and status_host.numel() < n:
        raise ValueError("status_host must hold >= n bytes")
    code = dtype_code(z_host.dtype, plain, eft)
    s_h2d, s_cmp, s_d2h = (ctypes.c_void_p(s.cuda_stream) for s in streams)
    rc = lib().polsar_inv_det_host(_ptr(z_host), _ptr(out_host), _ptr(status_host), n, ld, code,
                                   int(algo), _ptr(workspace),
                                   workspace.numel() * workspace.element_size(), s_h2d, s_cmp, s_d2h)
    check(rc, "polsar_inv_det_host")
    return out_host
