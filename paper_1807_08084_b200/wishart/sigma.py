"""Population covariance tables Sigma for the BASELINE configs (support).

Each table row is the lower-triangular Cholesky factor C of one Sigma
(Sigma = C C^H), 9 doubles: c00, Re c10, Im c10, c11, Re c20, Im c20, Re c21,
Im c21, c22 -- the layout wishart_core.h consumes.  Everything is built on the
host in fp64 with elementwise numpy arithmetic (Gram-Schmidt, 3x3 Cholesky),
from a numpy PCG64 stream keyed by (seed, stream id, tag), so a table depends
only on its key and its row count.  Laws:

  single     BASELINE configs[0]: Sigma = [[1, .3+.1i, .2], [.3-.1i, .5, .05i], [.2, -.05i, .8]]
  random     configs[1] / [4]: Sigma = A A^H / 3 + 0.1 I, A iid CN(0, 1)
  per-row    configs[2] / [3]: Sigma_r = U diag(1, k^u, k) U^H, U Haar,
             k log-uniform on [1, 1e3], u ~ U(0, 1)  (kappa_2(Sigma_r) = k <= 1e3)
"""
from __future__ import annotations

import numpy as np

SIGMA_C1 = np.array([[1.0, 0.3 + 0.1j, 0.2],
                     [0.3 - 0.1j, 0.5, 0.05j],
                     [0.2, -0.05j, 0.8]], dtype=np.complex128)


def _rng(seed: int, stream: int, tag: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, stream, tag])))


def _cn(rng, shape):
    """Circular complex normal CN(0, 1): Re, Im iid N(0, 1/2)."""
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) * np.sqrt(0.5)


def cholesky_table(sig: np.ndarray) -> np.ndarray:
    """(n, 3, 3) Hermitian PD -> (n, 9) lower Cholesky factors (elementwise).

    Real arithmetic only: numpy's complex division and multiplication take
    different SIMD / tail paths by array length, so a row's factor could
    depend on how many rows the table has; real ufuncs are one correctly
    rounded IEEE operation per element, whatever the length."""
    sig = np.asarray(sig, dtype=np.complex128).reshape(-1, 3, 3)
    s00, s11, s22 = sig[:, 0, 0].real, sig[:, 1, 1].real, sig[:, 2, 2].real
    s10r, s10i = sig[:, 1, 0].real, sig[:, 1, 0].imag
    s20r, s20i = sig[:, 2, 0].real, sig[:, 2, 0].imag
    s21r, s21i = sig[:, 2, 1].real, sig[:, 2, 1].imag
    c00 = np.sqrt(s00)
    c10r, c10i = s10r / c00, s10i / c00
    c20r, c20i = s20r / c00, s20i / c00
    c11 = np.sqrt(s11 - (c10r * c10r + c10i * c10i))
    # c21 = (s21 - c20 conj(c10)) / c11
    c21r = (s21r - (c20r * c10r + c20i * c10i)) / c11
    c21i = (s21i - (c20i * c10r - c20r * c10i)) / c11
    c22 = np.sqrt(s22 - (c20r * c20r + c20i * c20i) - (c21r * c21r + c21i * c21i))
    if not (np.all(np.isfinite(c11)) and np.all(np.isfinite(c22)) and np.all(c22 > 0)):
        raise ValueError("Sigma is not positive definite")
    return np.stack([c00, c10r, c10i, c11, c20r, c20i, c21r, c21i, c22], axis=1).astype(np.float64)


def sigma_from_table(tab: np.ndarray) -> np.ndarray:
    """Inverse of cholesky_table: (n, 9) -> (n, 3, 3) Sigma = C C^H."""
    tab = np.asarray(tab, dtype=np.float64).reshape(-1, 9)
    n = tab.shape[0]
    c = np.zeros((n, 3, 3), dtype=np.complex128)
    c[:, 0, 0] = tab[:, 0]
    c[:, 1, 0] = tab[:, 1] + 1j * tab[:, 2]
    c[:, 1, 1] = tab[:, 3]
    c[:, 2, 0] = tab[:, 4] + 1j * tab[:, 5]
    c[:, 2, 1] = tab[:, 6] + 1j * tab[:, 7]
    c[:, 2, 2] = tab[:, 8]
    return c @ np.conj(np.transpose(c, (0, 2, 1)))


def random_hpd(k: int, seed: int, stream: int) -> np.ndarray:
    """k matrices A A^H / 3 + 0.1 I with A iid CN(0, 1) (configs[1], [4])."""
    a = _cn(_rng(seed, stream, 1), (k, 3, 3))
    return a @ np.conj(np.transpose(a, (0, 2, 1))) / 3.0 + 0.1 * np.eye(3)


def haar_unitary(n: int, rng) -> np.ndarray:
    """n Haar unitaries by Gram-Schmidt of CN(0, I) columns (elementwise)."""
    v = _cn(rng, (n, 3, 3))  # v[:, :, k] = column k
    q = np.empty_like(v)
    for k in range(3):
        w = v[:, :, k].copy()
        for j in range(k):
            proj = np.sum(np.conj(q[:, :, j]) * w, axis=1)
            w = w - proj[:, None] * q[:, :, j]
        nrm = np.sqrt(np.sum(w.real * w.real + w.imag * w.imag, axis=1))
        q[:, :, k] = w / nrm[:, None]
    return q


PER_ROW_BLOCK = 1024


def per_row(rows: int, seed: int, stream: int, kappa_max: float = 1e3) -> np.ndarray:
    """Sigma_r = U diag(1, k^u, k) U^H for r < rows (configs[2], [3]).

    Prefix-stable: rows are drawn in blocks of PER_ROW_BLOCK, block b from its
    own PCG64 stream keyed by (seed, stream id, tag, b), so row r's Sigma
    depends only on (seed, stream, r) -- per_row(h)[:m] == per_row(m) for any
    m <= h.  An N-GPU image of N x H rows (weak scaling) therefore starts with
    the 1-GPU image, and a pixel's input never depends on the image height."""
    blocks = []
    for b in range((rows + PER_ROW_BLOCK - 1) // PER_ROW_BLOCK):
        rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, stream, 2, b])))
        u_haar = haar_unitary(PER_ROW_BLOCK, rng)
        kap = np.exp(rng.uniform(0.0, 1.0, PER_ROW_BLOCK) * np.log(kappa_max))
        u = rng.uniform(0.0, 1.0, PER_ROW_BLOCK)
        lam = np.stack([np.ones(PER_ROW_BLOCK), kap ** u, kap], axis=1)
        blocks.append((u_haar * lam[:, None, :]) @ np.conj(np.transpose(u_haar, (0, 2, 1))))
    if not blocks:
        return np.zeros((0, 3, 3), dtype=np.complex128)
    return np.concatenate(blocks)[:rows]
