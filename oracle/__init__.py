"""CPU oracle for arXiv 1807.08084 -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product package ``paper_1807_08084_b200`` never imports it, and the two share
no code (see ``polsar_oracle.c``'s header for what each function follows and
what pins it).

The arithmetic lives in ``polsar_oracle.c`` (binary128 / long double, plain
definitions);
this module only marshals numpy arrays through ctypes, plus two library-
primitive helpers (numpy ``eigvalsh`` for kappa_2, dense complex matmul for
the residual) that tests use as independent checks.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "polsar_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

# Plane order of the packed Hermitian matrix (PAPER.md:136-153 [§II-A]).
FIELDS = ("a", "re_b", "im_b", "re_c", "im_c", "d", "re_e", "im_e", "f")


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C, -O2, no fast-math, no FMA
    contraction so the extended-precision arithmetic is evaluated as
    written; binary128 through libquadmath)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off",
               "-fno-fast-math", _SRC, "-o", _LIB + ".tmp", "-lquadmath", "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def _host_tag() -> str:
    """-march=native code is only valid on the CPU it was built for: the plain
    build's file name carries a hash of this host's CPU model and flags (the
    repo travels between the build container and the GPU boxes)."""
    import hashlib
    try:
        with open("/proc/cpuinfo") as f:
            lines = [l for l in f if l.startswith(("model name", "flags"))][:2]
    except OSError:
        lines = ["unknown"]
    return hashlib.sha1("".join(lines).encode()).hexdigest()[:12]


def build_plain(force: bool = False) -> str:
    """The same source optimised for speed (-O3 -march=native, FMA contraction
    allowed): the storage-precision entry points oracle_inv_det_plain_* are
    SURVEY §8(d)'s plain CPU baseline.  Never used for verification."""
    out = os.path.join(_HERE, f"liboracle_plain_{_host_tag()}.so")
    if force or not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(_SRC):
        tmp = f"{out}.{os.getpid()}.tmp"
        cmd = ["gcc", "-O3", "-march=native", "-std=gnu11", "-fPIC", "-shared", _SRC,
               "-o", tmp, "-lquadmath", "-lm"]
        subprocess.check_call(cmd)
        os.replace(tmp, out)
    return out


_lib = None
_lib_plain = None
_lib_lock = threading.Lock()


def lib() -> ctypes.CDLL:
    """The loaded oracle library with its signatures declared.  Published only
    once fully configured (the *_threaded helpers call it from many threads)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        _lib_new = ctypes.CDLL(build())
        _configure(_lib_new)
        _lib = _lib_new
    return _lib


def lib_plain() -> ctypes.CDLL:
    global _lib_plain
    if _lib_plain is not None:
        return _lib_plain
    with _lib_lock:
        if _lib_plain is None:
            lp = ctypes.CDLL(build_plain())
            P, I64 = ctypes.c_void_p, ctypes.c_int64
            lp.oracle_inv_det_plain_s.argtypes = [P, I64, P, I64, I64]
            lp.oracle_inv_det_plain_d.argtypes = [P, I64, P, I64, I64]
            _lib_plain = lp
    return _lib_plain


def inv_det_plain(z: np.ndarray, threads: int = 1, out: np.ndarray | None = None) -> np.ndarray:
    """The cofactor definition in the storage precision (float for float32
    input, double for float64), columns split over `threads` host threads:
    SURVEY §8(d)'s plain CPU baseline (-O3 -march=native build).  Returns
    (11, n) in the input dtype (into `out` when given: a reused, already
    touched buffer keeps first-touch page faults out of a timing).  For
    timing, not for verification."""
    z = _planes(z)
    n = z.shape[1]
    if out is None:
        out = np.empty((11, n), dtype=z.dtype)
    if out.shape != (11, n) or out.dtype != z.dtype or not out.flags.c_contiguous:
        raise ValueError("out must be a contiguous (11, n) array of z's dtype")
    lp = lib_plain()
    fn = lp.oracle_inv_det_plain_s if z.dtype == np.float32 else lp.oracle_inv_det_plain_d
    esz = z.itemsize
    if threads <= 1:
        fn(_ptr(z), n, _ptr(out), n, n)
        return out
    bounds = np.linspace(0, n, threads + 1).astype(np.int64)

    def work(k):
        lo, hi = int(bounds[k]), int(bounds[k + 1])
        if hi > lo:
            fn(_ptr(z) + lo * esz, n, _ptr(out) + lo * esz, n, hi - lo)

    with ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(work, range(threads)))
    return out


def _configure(_lib: ctypes.CDLL) -> None:
    P, I64, D, INT = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int
    _lib.oracle_inv_det_plain_s.argtypes = [P, I64, P, I64, I64]
    _lib.oracle_inv_det_plain_d.argtypes = [P, I64, P, I64, I64]
    _lib.oracle_inv_det_f64.argtypes = [P, I64, P, I64, P, I64]
    _lib.oracle_inv_det_f32.argtypes = [P, I64, P, I64, P, I64]
    _lib.oracle_gauss_jordan.argtypes = [P, P, P]
    _lib.oracle_gauss_jordan.restype = INT
    _lib.oracle_pair_distance.argtypes = [P, P, D]
    _lib.oracle_pair_distance.restype = D
    _lib.oracle_window_f64.argtypes = [P, I64, I64, I64, INT, D, D, P, I64, P]
    _lib.oracle_window_f32.argtypes = [P, I64, I64, I64, INT, D, D, P, I64, P]
    _lib.oracle_inv_det_blocks_f64.argtypes = [P, I64, INT, P, I64, I64]
    _lib.oracle_inv_det_blocks_f32.argtypes = [P, I64, INT, P, I64, I64]
    _lib.oracle_nlm_f64.argtypes = [P, I64, I64, I64, INT, D, D, P, I64, P]
    _lib.oracle_nlm_f32.argtypes = [P, I64, I64, I64, INT, D, D, P, I64, P]
    _lib.oracle_window_kl_f64.argtypes = [P, I64, I64, I64, INT, D, D, P, I64, P]
    _lib.oracle_window_kl_f32.argtypes = [P, I64, I64, I64, INT, D, D, P, I64, P]
    _lib.oracle_kl_distance.argtypes = [P, P, D]
    _lib.oracle_kl_distance.restype = D
    _lib.oracle_ldbl_mant_dig.restype = INT
    _lib.oracle_quad_mant_dig.restype = INT


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _planes(z: np.ndarray) -> np.ndarray:
    z = np.asarray(z)
    if z.ndim != 2 or z.shape[0] != 9:
        raise ValueError("z must have shape (9, n)")
    if z.dtype not in (np.float32, np.float64):
        raise TypeError("z must be float32 or float64")
    return np.ascontiguousarray(z)


def inv_det(z: np.ndarray, with_imag: bool = False):
    """Z^-1 (9 planes), det Z, det Z^-1 for every column of z (shape (9, n)).

    Returns a float64 array of shape (11, n) (planes 0..8 inverse in FIELDS
    order, 9 det, 10 1/det); with ``with_imag`` also Im of the Eq. (5)
    expansion.  Cofactor expansion (Eq. 3-5), binary128, one final rounding.
    """
    z = _planes(z)
    n = z.shape[1]
    out = np.empty((11, n), dtype=np.float64)
    im = np.empty(n, dtype=np.float64) if with_imag else None
    fn = lib().oracle_inv_det_f64 if z.dtype == np.float64 else lib().oracle_inv_det_f32
    fn(_ptr(z), n, _ptr(out), n, _ptr(im) if im is not None else None, n)
    return (out, im) if with_imag else out


def inv_det_blocks(z: np.ndarray, nblocks: int) -> np.ndarray:
    """Multi-frequency block-diagonal pixels: z has
    9*nblocks planes; returns (9*nblocks + 2, n) -- block inverses, det and
    det^-1 of the whole block-diagonal matrix (binary128, blockwise cofactor
    definition, products of the block determinants)."""
    z = np.ascontiguousarray(np.asarray(z))
    if z.ndim != 2 or z.shape[0] != 9 * nblocks:
        raise ValueError("z must have shape (9*nblocks, n)")
    n = z.shape[1]
    out = np.empty((9 * nblocks + 2, n), dtype=np.float64)
    fn = lib().oracle_inv_det_blocks_f64 if z.dtype == np.float64 else lib().oracle_inv_det_blocks_f32
    fn(_ptr(z), n, int(nblocks), _ptr(out), n, n)
    return out


def inv_det_threaded(z: np.ndarray, threads: int) -> np.ndarray:
    """Same as :func:`inv_det`, the columns split over ``threads`` host
    threads (ctypes drops the GIL during the foreign call).  Used only to time
    the oracle as a CPU baseline."""
    z = _planes(z)
    n = z.shape[1]
    out = np.empty((11, n), dtype=np.float64)
    fn = lib().oracle_inv_det_f64 if z.dtype == np.float64 else lib().oracle_inv_det_f32
    esz = z.itemsize
    bounds = np.linspace(0, n, threads + 1).astype(np.int64)

    def work(k):
        lo, hi = int(bounds[k]), int(bounds[k + 1])
        if hi > lo:
            fn(_ptr(z) + lo * esz, n, _ptr(out) + lo * 8, n, None, hi - lo)

    with ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(work, range(threads)))
    return out


def to_full(z: np.ndarray) -> np.ndarray:
    """Packed (9, n) -> full complex (n, 3, 3) Hermitian matrices (layout of
    PAPER.md:136-153)."""
    z = np.asarray(z, dtype=np.float64)
    a, br, bi, cr, ci, d, er, ei, f = z
    b, c, e = br + 1j * bi, cr + 1j * ci, er + 1j * ei
    n = z.shape[1]
    m = np.empty((n, 3, 3), dtype=np.complex128)
    m[:, 0, 0], m[:, 0, 1], m[:, 0, 2] = a, b, c
    m[:, 1, 0], m[:, 1, 1], m[:, 1, 2] = np.conj(b), d, e
    m[:, 2, 0], m[:, 2, 1], m[:, 2, 2] = np.conj(c), np.conj(e), f
    return m


def gauss_jordan(z: np.ndarray):
    """Brute force: full inverse (n, 3, 3) and complex det (n,) by complex
    Gauss-Jordan with partial pivoting on the full matrix (tiny inputs)."""
    full = to_full(z)
    n = full.shape[0]
    inv = np.empty((n, 3, 3), dtype=np.complex128)
    det = np.empty(n, dtype=np.complex128)
    m18 = np.empty(18, dtype=np.float64)
    i18 = np.empty(18, dtype=np.float64)
    d2 = np.empty(2, dtype=np.float64)
    for k in range(n):
        m18[0::2] = full[k].real.ravel()
        m18[1::2] = full[k].imag.ravel()
        rc = lib().oracle_gauss_jordan(_ptr(m18), _ptr(i18), _ptr(d2))
        if rc:
            inv[k] = np.nan
            det[k] = 0.0
            continue
        inv[k] = (i18[0::2] + 1j * i18[1::2]).reshape(3, 3)
        det[k] = d2[0] + 1j * d2[1]
    return inv, det


def pair_distance(zi: np.ndarray, zj: np.ndarray, looks: float) -> float:
    """d_ij = L [ln det((Z_i+Z_j)/2) - (ln det Z_i + ln det Z_j)/2]."""
    zi = np.ascontiguousarray(zi, dtype=np.float64).reshape(9)
    zj = np.ascontiguousarray(zj, dtype=np.float64).reshape(9)
    return lib().oracle_pair_distance(_ptr(zi), _ptr(zj), float(looks))


def window(z: np.ndarray, height: int, width: int, radius: int, looks: float,
           h: float, idx=None) -> np.ndarray:
    """W_i = sum over the clipped (2R+1)^2 window of exp(-d_ij/h) for the
    pixels ``idx`` (row-major indices; all pixels if None)."""
    z = _planes(z)
    if z.shape[1] < height * width:
        raise ValueError("z has fewer than height*width pixels")
    if idx is None:
        idx = np.arange(height * width, dtype=np.int64)
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    out = np.empty(idx.shape[0], dtype=np.float64)
    fn = lib().oracle_window_f64 if z.dtype == np.float64 else lib().oracle_window_f32
    fn(_ptr(z), z.shape[1], height, width, int(radius), float(looks), float(h),
       _ptr(idx), idx.shape[0], _ptr(out))
    return out


def kl_distance(zi, zj, looks: float) -> float:
    """Symmetric Wishart KL distance L[(tr(Zi^-1 Zj) + tr(Zj^-1 Zi))/2 - 3]."""
    zi = np.ascontiguousarray(zi, dtype=np.float64).reshape(9)
    zj = np.ascontiguousarray(zj, dtype=np.float64).reshape(9)
    return lib().oracle_kl_distance(_ptr(zi), _ptr(zj), float(looks))


def window_kl(z, height, width, radius, looks, h, idx=None):
    """W_i with the symmetric Wishart KL distance (long double)."""
    z = _planes(z)
    if idx is None:
        idx = np.arange(height * width, dtype=np.int64)
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    out = np.empty(idx.shape[0], dtype=np.float64)
    fn = lib().oracle_window_kl_f64 if z.dtype == np.float64 else lib().oracle_window_kl_f32
    fn(_ptr(z), z.shape[1], height, width, int(radius), float(looks), float(h), _ptr(idx),
       idx.shape[0], _ptr(out))
    return out


def window_kl_threaded(z, height, width, radius, looks, h, idx, threads):
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    parts = [p for p in np.array_split(idx, threads) if p.size]
    with ThreadPoolExecutor(max_workers=threads) as ex:
        res = list(ex.map(lambda p: window_kl(z, height, width, radius, looks, h, p), parts))
    return np.concatenate(res)


def nlm(z: np.ndarray, height: int, width: int, radius: int, looks: float, h: float, idx=None):
    """NLM filter output: returns (Zhat (9, m), W (m,)) for pixels idx,
    Zhat_i = sum_j w_ij Z_j / W_i with the window weights (long double)."""
    z = _planes(z)
    if idx is None:
        idx = np.arange(height * width, dtype=np.int64)
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    m = idx.shape[0]
    out = np.empty((10, m), dtype=np.float64)
    fn = lib().oracle_nlm_f64 if z.dtype == np.float64 else lib().oracle_nlm_f32
    fn(_ptr(z), z.shape[1], height, width, int(radius), float(looks), float(h), _ptr(idx), m,
       _ptr(out))
    return out[:9], out[9]


def nlm_threaded(z, height, width, radius, looks, h, idx, threads):
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    parts = [p for p in np.array_split(idx, threads) if p.size]
    with ThreadPoolExecutor(max_workers=threads) as ex:
        res = list(ex.map(lambda p: nlm(z, height, width, radius, looks, h, p), parts))
    return np.concatenate([r[0] for r in res], axis=1), np.concatenate([r[1] for r in res])


def window_threaded(z, height, width, radius, looks, h, idx, threads):
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    parts = np.array_split(idx, threads)
    with ThreadPoolExecutor(max_workers=threads) as ex:
        res = list(ex.map(lambda p: window(z, height, width, radius, looks, h, p)
                          if p.size else np.empty(0), parts))
    return np.concatenate(res)


def kappa2(z: np.ndarray) -> np.ndarray:
    """Spectral condition number lambda_max / lambda_min of each matrix
    (numpy/LAPACK eigvalsh on the full Hermitian matrix; library primitive).
    Non-positive lambda_min gives inf."""
    w = np.linalg.eigvalsh(to_full(z))
    lo, hi = w[:, 0], w[:, 2]
    with np.errstate(divide="ignore", invalid="ignore"):
        k = np.where(lo > 0, hi / lo, np.inf)
    return k


def residual(z: np.ndarray, inv9: np.ndarray) -> np.ndarray:
    """max |Z * Z^-1 - I| per matrix by an independent dense complex multiply
    of the full matrices (the inverse's lower triangle rebuilt by Hermitian
    symmetry)."""
    prod = to_full(z) @ to_full(inv9)
    prod -= np.eye(3)[None]
    return np.abs(prod).reshape(prod.shape[0], -1).max(axis=1)


def ldbl_mant_dig() -> int:
    return lib().oracle_ldbl_mant_dig()


def quad_mant_dig() -> int:
    return lib().oracle_quad_mant_dig()
