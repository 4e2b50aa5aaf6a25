"""Exact rational arithmetic for pinning the oracle (test helper).

Every IEEE double is a rational number, so the exact inverse and determinant
of a matrix of doubles can be computed with ``fractions.Fraction`` over the
Gaussian rationals Q(i).  This is Gauss-Jordan elimination on the full 3x3
matrix -- no cofactors, no Hermitian packing -- so it shares nothing with the
oracle's cofactor expansion (Eq. 3-5) it is used to check.
"""
from __future__ import annotations

from fractions import Fraction


class QI:
    """a + b i with a, b rational."""

    __slots__ = ("re", "im")

    def __init__(self, re, im=0):
        self.re = Fraction(re)
        self.im = Fraction(im)

    def __add__(self, o):
        return QI(self.re + o.re, self.im + o.im)

    def __sub__(self, o):
        return QI(self.re - o.re, self.im - o.im)

    def __mul__(self, o):
        return QI(self.re * o.re - self.im * o.im, self.re * o.im + self.im * o.re)

    def conj(self):
        return QI(self.re, -self.im)

    def inv(self):
        den = self.re * self.re + self.im * self.im
        return QI(self.re / den, -self.im / den)

    def is_zero(self):
        return self.re == 0 and self.im == 0


def full_from_packed(p9):
    """Packed (a, re b, im b, re c, im c, d, re e, im e, f) -> 3x3 of QI."""
    a, br, bi, cr, ci, d, er, ei, f = (Fraction(float(x)) for x in p9)
    b, c, e = QI(br, bi), QI(cr, ci), QI(er, ei)
    return [[QI(a), b, c], [b.conj(), QI(d), e], [c.conj(), e.conj(), QI(f)]]


def exact_inverse_det(p9):
    """Exact (inverse 3x3 of QI, det QI) by Gauss-Jordan over Q(i)."""
    m = full_from_packed(p9)
    aug = [row[:] + [QI(1 if k == r else 0) for k in range(3)] for r, row in enumerate(m)]
    det = QI(1)
    for col in range(3):
        piv = next((r for r in range(col, 3) if not aug[r][col].is_zero()), None)
        if piv is None:
            return None, QI(0)
        if piv != col:
            aug[col], aug[piv] = aug[piv], aug[col]
            det = QI(-det.re, -det.im)
        pv = aug[col][col]
        det = det * pv
        pinv = pv.inv()
        aug[col] = [x * pinv for x in aug[col]]
        for r in range(3):
            if r != col and not aug[r][col].is_zero():
                fct = aug[r][col]
                aug[r] = [x - fct * y for x, y in zip(aug[r], aug[col])]
    inv = [row[3:] for row in aug]
    return inv, det


def packed_upper(inv):
    """Upper triangle of a 3x3 QI matrix in the packed field order, as floats
    (each rounded once from the exact rational)."""
    return [float(inv[0][0].re), float(inv[0][1].re), float(inv[0][1].im),
            float(inv[0][2].re), float(inv[0][2].im), float(inv[1][1].re),
            float(inv[1][2].re), float(inv[1][2].im), float(inv[2][2].re)]
