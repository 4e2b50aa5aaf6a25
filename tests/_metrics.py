"""Error metrics shared by the parity tests (reading R-10).

Per pixel:
  inverse  normwise  max_k |got_k - ref_k| / max_k |ref_k| over the 9 reals
  det, 1/det         |got - ref| / |ref|
BASELINE's tolerance (max relative error <= 1e-12 fp64, <= 2e-5 fp32) is
asserted over pixels whose oracle kappa_2 <= 1e4; the rest are reported.
"""
import numpy as np

TOL = {"float64": 1e-12, "float32": 2e-5}


def errors(got, ref):
    got = np.asarray(got, dtype=np.float64)
    inv = np.max(np.abs(got[:9] - ref[:9]), axis=0) / np.max(np.abs(ref[:9]), axis=0)
    det = np.abs(got[9] - ref[9]) / np.abs(ref[9])
    idet = np.abs(got[10] - ref[10]) / np.abs(ref[10])
    return inv, det, idet


def entrywise(got, ref):
    """Per complex entry relative error |Δ entry| / |entry| (reported)."""
    got = np.asarray(got, dtype=np.float64)
    out = []
    for idx in ([0], [1, 2], [3, 4], [5], [6, 7], [8]):
        d = np.sqrt(np.sum((got[idx] - ref[idx]) ** 2, axis=0))
        m = np.sqrt(np.sum(ref[idx] ** 2, axis=0))
        with np.errstate(divide="ignore", invalid="ignore"):
            out.append(np.where(m > 0, d / m, 0.0))
    return np.max(np.stack(out), axis=0)


def worst(got, ref, mask):
    inv, det, idet = errors(got, ref)
    return float(max(inv[mask].max(initial=0), det[mask].max(initial=0), idet[mask].max(initial=0)))


def status_expected(z, ref, storage):
    """Status the kernels must report, decided from the oracle's exact det:
    SINGULAR (1) iff det <= tau a d f, tau = 16 u_in (R-5).
    Returns (expected, decidable) -- pixels within 1e-6 relative of the
    threshold are not decidable across precisions and are excluded."""
    u = 2.0 ** -24 if storage == "float32" else 2.0 ** -53
    z = np.asarray(z, dtype=np.float64)
    thr = 16 * u * z[0] * z[5] * z[8]
    det = ref[9]
    expected = np.where(det > thr, 0, 1).astype(np.uint8)
    decidable = np.abs(det - thr) > 1e-6 * np.abs(thr)
    return expected, decidable
