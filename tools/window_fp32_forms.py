"""Numerical experiment (CPU, numpy): how accurate is the window sum W_i
(R-12) when the pair determinant det(Z_i + Z_j) is taken in
fp32, in two forms?

  direct:  S = fl32(Z_i + Z_j), det S by Eq. 6 in fp32 (the kernel's plain mode)
  mixed:   det(A + B) = det A + det B + tr(adj(A) B) + tr(A adj(B))  (3x3
           identity; with A, B Hermitian PD every term is positive), adj and
           det per pixel in fp64 rounded once to fp32, the two traces as
           9-term fp32 dot products

against W in fp64.  numpy's float32 has no FMA, so this bounds the kernel's
fp32 arithmetic loosely.  Usage: python tools/window_fp32_forms.py [rows]
"""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_1807_08084_b200 import configs, wishart  # noqa: E402


def det6(a, br, bi, cr, ci, d, er, ei, f):
    ac = d * f - (er * er + ei * ei)
    bcr = cr * er + ci * ei - br * f
    bci = ci * er - (cr * ei + bi * f)
    ccr = br * er - (bi * ei + cr * d)
    cci = br * ei + bi * er - ci * d
    return a * ac + br * bcr + bi * bci + cr * ccr + ci * cci


def adj_planes(z):
    """adj(Z) of Hermitian [[a, b, c], [b*, d, e], [c*, e*, f]] as
    (A00, A11, A22, A01r, A01i, A02r, A02i, A12r, A12i), in fp64."""
    a, br, bi, cr, ci, d, er, ei, f = z
    b, c, e = br + 1j * bi, cr + 1j * ci, er + 1j * ei
    A00 = d * f - np.abs(e) ** 2
    A11 = a * f - np.abs(c) ** 2
    A22 = a * d - np.abs(b) ** 2
    A01 = c * np.conj(e) - b * f        # cofactor transpose entries
    A02 = b * e - c * d
    A12 = np.conj(b) * c - a * e
    return np.stack([A00, A11, A22, A01.real, A01.imag, A02.real, A02.imag, A12.real, A12.imag])


def tr_prod(X, Z):
    """tr(X Z) = sum_k X_kk Z_kk + 2 sum_{k<l} Re(X_kl conj(Z_kl)) for Hermitian X, Z."""
    a, br, bi, cr, ci, d, er, ei, f = Z
    two = X.dtype.type(2)
    return (X[0] * a + X[1] * d + X[2] * f
            + two * (X[3] * br + X[4] * bi) + two * (X[5] * cr + X[6] * ci)
            + two * (X[7] * er + X[8] * ei))


def main():
    rows = int(sys.argv[1]) if len(sys.argv) > 1 else 96
    cfg = configs.get("c5")
    R, w = cfg.radius, cfg.width
    z = wishart.generate_cpu(cfg, 0, rows).astype(np.float32).reshape(9, rows, w)
    z64 = z.astype(np.float64)
    det64 = det6(*z64)
    adj64 = adj_planes(z64)
    # check the identity on fp64 against the direct det (sanity)
    s = z64[:, :, :-1] + z64[:, :, 1:]
    lhs = det6(*s)
    rhs = det64[:, :-1] + det64[:, 1:] + tr_prod(adj64[:, :, :-1], z64[:, :, 1:]) + tr_prod(adj64[:, :, 1:], z64[:, :, :-1])
    print("identity rel err (fp64):", float(np.max(np.abs(lhs - rhs) / lhs)))
    g64 = 1.0 / (8.0 * det64)
    z32, det32, adj32, g32 = z, det64.astype(np.float32), adj64.astype(np.float32), g64.astype(np.float32)
    W = {k: np.zeros((rows, w)) for k in ("f64", "direct", "mixed")}
    for dy in range(-R, R + 1):
        for dx in range(-R, R + 1):
            ys, ye = max(0, -dy), min(rows, rows - dy)
            xs, xe = max(0, -dx), min(w, w - dx)
            I = (slice(None), slice(ys, ye), slice(xs, xe))
            J = (slice(None), slice(ys + dy, ye + dy), slice(xs + dx, xe + dx))
            Ii, Jj = I[1:], J[1:]
            ds = det6(*(z64[I] + z64[J]))
            rr = (ds * g64[Ii]) * (ds * g64[Jj])
            W["f64"][Ii] += 1.0 / (rr * rr)
            ds = det6(*(z32[I] + z32[J]))
            rr = (ds * g32[Ii]) * (ds * g32[Jj])
            W["direct"][Ii] += (np.float32(1) / (rr * rr)).astype(np.float64)
            ds = (det32[Ii] + det32[Jj]) + (tr_prod(adj32[I], z32[J]) + tr_prod(adj32[J], z32[I]))
            rr = (ds * g32[Ii]) * (ds * g32[Jj])
            W["mixed"][Ii] += (np.float32(1) / (rr * rr)).astype(np.float64)
    for k in ("direct", "mixed"):
        e = np.abs(W[k] - W["f64"]) / W["f64"]
        print(f"{k:7s} max rel err {e.max():.3e}  p99.9 {np.quantile(e, 0.999):.3e}  mean {e.mean():.3e}")


if __name__ == "__main__":
    main()
