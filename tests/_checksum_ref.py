"""Independent numpy evaluation of the R1 output checksum (
include/polsar.h `polsar_checksum`): for pixel p (global index pix_offset + p)
and plane k,

    h += mix64(bits(plane_k[p]) XOR (key(p) + k * 0xD6E8FEB86659FD93)),
    key(p) = (pix_offset + p) * 0x9E3779B97F4A7C15   (mod 2^64),

summed with wrapping uint64 addition (order-independent), and the status
counts are a plain ``bincount`` of the status plane.  mix64 is the SplitMix64
finaliser.  Written from that definition with vectorised numpy uint64
arithmetic; it shares nothing with csrc/checksum.cu.
"""
import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_PLANE = np.uint64(0xD6E8FEB86659FD93)


def mix64(x):
    x = np.asarray(x, dtype=np.uint64).copy()
    with np.errstate(over="ignore"):
        x ^= x >> np.uint64(30)
        x *= np.uint64(0xbf58476d1ce4e5b9)
        x ^= x >> np.uint64(27)
        x *= np.uint64(0x94d049bb133111eb)
        x ^= x >> np.uint64(31)
    return x


def checksum(planes, pix_offset=0, status=None, chunk=1 << 22):
    """planes: (nplanes, n) float32 or float64 numpy array (bit patterns are
    hashed, zero-extended to 64 bits for float32).  Returns (hash, [n_ok,
    n_singular, n_not_pd]) as Python ints."""
    planes = np.ascontiguousarray(planes)
    nplanes, n = planes.shape
    ubits = planes.view(np.uint32 if planes.dtype == np.float32 else np.uint64)
    h = np.uint64(0)
    with np.errstate(over="ignore"):
        for lo in range(0, n, chunk):
            hi = min(n, lo + chunk)
            key = (np.arange(lo, hi, dtype=np.uint64) + np.uint64(pix_offset)) * _GOLDEN
            for k in range(nplanes):
                v = ubits[k, lo:hi].astype(np.uint64)
                h += mix64(v ^ (key + np.uint64(k) * _PLANE)).sum(dtype=np.uint64)
    counts = [0, 0, 0]
    if status is not None:
        bc = np.bincount(np.asarray(status, dtype=np.uint8), minlength=3)
        counts = [int(bc[0]), int(bc[1]), int(bc[2])]
    return int(h), counts
