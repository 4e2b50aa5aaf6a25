"""Pins for the CPU oracle (``-m "not gpu"``).

The oracle (oracle/polsar_oracle.c) is the plain definition of Z^-1, det Z and
det Z^-1 (Eq. 3-5) and of the window sum (BASELINE configs[4]).  Each
test below checks it against something other than itself: hand-derived worked
examples, exact rational arithmetic, a brute-force Gauss-Jordan, LAPACK, closed
forms and invariants.  A dropped term, a wrong sign / index / conjugation or a
transposed operand in the oracle fails at least the exact-rational test and
the Z*Z^-1 = I residual test.
"""
import math
import os

import numpy as np
import pytest

import oracle
from tests._exact import exact_inverse_det, packed_upper

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "worked_examples.txt")


def rand_hpd(n, seed, ridge=0.1, scale_spread=False):
    """Test-local random HPD matrices G G^H / 3 + ridge I (packed, float64)."""
    rng = np.random.default_rng(seed)
    g = (rng.standard_normal((n, 3, 3)) + 1j * rng.standard_normal((n, 3, 3))) / math.sqrt(2)
    m = g @ np.conj(np.transpose(g, (0, 2, 1))) / 3 + ridge * np.eye(3)
    if scale_spread:
        m *= np.exp(rng.uniform(-10, 10, n))[:, None, None]
    return pack(m)


def pack(m):
    return np.stack([m[:, 0, 0].real, m[:, 0, 1].real, m[:, 0, 1].imag,
                     m[:, 0, 2].real, m[:, 0, 2].imag, m[:, 1, 1].real,
                     m[:, 1, 2].real, m[:, 1, 2].imag, m[:, 2, 2].real]).astype(np.float64)


def rand_kappa(n, seed, kappa):
    """U diag(1, k^u, k) U^H with U Haar (numpy QR, phase-fixed): kappa_2 = k."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, 3, 3)) + 1j * rng.standard_normal((n, 3, 3))
    q, r = np.linalg.qr(x)
    ph = np.diagonal(r, axis1=1, axis2=2)
    q = q * (ph / np.abs(ph))[:, None, :]
    u = rng.uniform(0, 1, n)
    lam = np.stack([np.ones(n), kappa ** u, np.full(n, float(kappa))], axis=1)
    m = (q * lam[:, None, :]) @ np.conj(np.transpose(q, (0, 2, 1)))
    return pack(m)


def normwise(got9, ref9):
    return np.max(np.abs(got9 - ref9), axis=0) / np.max(np.abs(ref9), axis=0)


def parse_golden():
    rows = []
    for line in open(GOLDEN):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        name, zin, inv, det, idet = [s.strip() for s in line.split("|")]
        rows.append((name, np.array(zin.split(), float), np.array(inv.split(), float),
                     float(det), float(idet)))
    return rows


def test_extended_precision():
    # the oracle must really evaluate in binary128 (inverse/det) and 80-bit
    # long double (window) on this host
    assert oracle.quad_mant_dig() == 113
    assert oracle.ldbl_mant_dig() == 64


@pytest.mark.parametrize("row", parse_golden(), ids=lambda r: r[0])
def test_worked_examples(row):
    name, zin, inv, det, idet = row
    out = oracle.inv_det(zin.reshape(9, 1))
    np.testing.assert_allclose(out[:9, 0], inv, rtol=0, atol=2e-16 * np.abs(inv).max())
    assert out[9, 0] == pytest.approx(det, rel=1e-16, abs=0)
    assert out[10, 0] == pytest.approx(idet, rel=2e-16, abs=0)
    if name in ("identity", "diag245", "golden"):
        # dyadic inputs with dyadic results: exact
        assert np.array_equal(out[:9, 0], inv)
        assert out[9, 0] == det and out[10, 0] == idet


def test_exact_rational_random():
    z = np.concatenate([rand_hpd(40, 1), rand_kappa(20, 2, 1e3)], axis=1)
    out = oracle.inv_det(z)
    for p in range(z.shape[1]):
        inv, det = exact_inverse_det(z[:, p])
        assert det.im == 0  # Hermitian => real determinant, exactly
        ref = np.array(packed_upper(inv))
        err = np.max(np.abs(out[:9, p] - ref)) / np.max(np.abs(ref))
        assert err <= 1e-15, (p, err)
        detf = float(det.re)
        # one final rounding (2^-53) plus binary128 rounding of the
        # expansion's terms, whose magnitude is bounded by 6 max|z|^3
        terms = 6 * np.max(np.abs(z[:, p])) ** 3
        bound = 1.2e-16 * abs(detf) + 32 * 2.0 ** -113 * terms
        assert abs(out[9, p] - detf) <= bound
        assert abs(out[10, p] - 1.0 / detf) <= 1.2e-16 / abs(detf) + bound / detf ** 2


def test_exact_rational_lower_triangle_hermitian():
    # the full exact inverse is Hermitian: the packed upper triangle determines it
    z = rand_hpd(10, 3)
    for p in range(z.shape[1]):
        inv, _ = exact_inverse_det(z[:, p])
        for r in range(3):
            for c in range(3):
                assert inv[r][c].re == inv[c][r].re and inv[r][c].im == -inv[c][r].im


def test_det_imag_vanishes():
    z = rand_hpd(5000, 4, scale_spread=True)
    out, im = oracle.inv_det(z, with_imag=True)
    scale = np.abs(z[0] * z[5] * z[8]) + np.abs(z).max(axis=0) ** 3
    assert np.all(np.abs(im) <= 64 * 2.0 ** -64 * scale)


def test_gauss_jordan_brute_force():
    z = np.concatenate([rand_hpd(3000, 5), rand_kappa(3000, 6, 1e6)], axis=1)
    out = oracle.inv_det(z)
    inv, det = oracle.gauss_jordan(z)
    k = oracle.kappa2(z)
    # the brute force's full inverse is Hermitian up to rounding
    herm = np.abs(inv - np.conj(np.transpose(inv, (0, 2, 1)))).max(axis=(1, 2))
    assert np.all(herm <= 1e-15 * k * np.abs(inv).max(axis=(1, 2)))
    gj9 = pack(inv)
    err = normwise(out[:9], gj9)
    assert np.all(err <= 1e-17 * k + 4e-16), err.max()
    assert np.all(np.abs(det.imag) <= 1e-15 * np.abs(det.real) * k)
    assert np.all(np.abs(out[9] - det.real) <= (1e-17 * k + 4e-16) * np.abs(det.real))


def test_lapack_special_case():
    z = rand_kappa(2000, 7, 1e4)
    out = oracle.inv_det(z)
    full = oracle.to_full(z)
    inv = np.linalg.inv(full)
    det = np.linalg.det(full)
    assert np.all(normwise(out[:9], pack(inv)) <= 1e-12)
    assert np.all(np.abs(out[9] - det.real) <= 1e-12 * np.abs(det.real))


def test_residual_identity():
    z = np.concatenate([rand_hpd(2000, 8), rand_kappa(2000, 9, 1e4)], axis=1)
    out = oracle.inv_det(z)
    k = oracle.kappa2(z)
    res = oracle.residual(z, out[:9])
    scale = np.abs(z).max(axis=0) * np.abs(out[:9]).max(axis=0)
    assert np.all(res <= 8 * 2.2e-16 * scale + 1e-18 * k * scale)


@pytest.mark.parametrize("m", [1, -3, 7])
def test_power_of_two_scaling_exact(m):
    z = rand_hpd(3000, 10, scale_spread=True)
    k = 2.0 ** m
    a = oracle.inv_det(z)
    b = oracle.inv_det(z * k)
    assert np.array_equal(b[:9], a[:9] / k)
    assert np.array_equal(b[9], a[9] * k ** 3)
    assert np.array_equal(b[10], a[10] / k ** 3)


def test_det_times_inverse_det():
    z = rand_hpd(5000, 11, scale_spread=True)
    out = oracle.inv_det(z)
    assert np.all(np.abs(out[9] * out[10] - 1.0) <= 4.5e-16)
    assert np.all(out[9] > 0)


def test_block_diagonal_closed_form():
    rng = np.random.default_rng(12)
    n = 1000
    a = rng.uniform(1, 3, n)
    d = rng.uniform(1, 3, n)
    f = rng.uniform(0.1, 2, n)
    b = rng.uniform(-0.7, 0.7, n) + 1j * rng.uniform(-0.7, 0.7, n)
    z = np.stack([a, b.real, b.imag, 0 * a, 0 * a, d, 0 * a, 0 * a, f])
    out = oracle.inv_det(z)
    g = a * d - np.abs(b) ** 2
    ref = np.stack([d / g, -b.real / g, -b.imag / g, 0 * a, 0 * a, a / g, 0 * a, 0 * a, 1 / f])
    assert np.all(normwise(out[:9], ref) <= 1e-15)
    np.testing.assert_allclose(out[9], g * f, rtol=1e-15)


def test_rank_one_is_singular():
    rng = np.random.default_rng(13)
    s = rng.standard_normal((500, 3)) + 1j * rng.standard_normal((500, 3))
    m = s[:, :, None] * np.conj(s[:, None, :])
    z = pack(m)
    out = oracle.inv_det(z)
    adf = z[0] * z[5] * z[8]
    assert np.all(np.abs(out[9]) <= 1e-15 * adf)


# ---------------------------------------------------------------- window oracle

def clipped_count(y, x, h, w, r):
    return (min(h - 1, y + r) - max(0, y - r) + 1) * (min(w - 1, x + r) - max(0, x - r) + 1)


def test_window_constant_image_exact():
    h, w, r = 9, 11, 3
    z0 = rand_hpd(1, 14)[:, 0]
    z = np.repeat(z0[:, None], h * w, axis=1)
    got = oracle.window(z, h, w, r, 4.0, 1.0)
    ref = np.array([clipped_count(p // w, p % w, h, w, r) for p in range(h * w)], float)
    assert np.array_equal(got, ref)


def test_window_two_class_closed_form():
    h, w, r, looks = 8, 10, 2, 4.0
    za, zb = rand_hpd(2, 15)[:, 0], rand_hpd(2, 15)[:, 1]
    xs = np.arange(h * w) % w
    z = np.where(xs[None, :] < 5, za[:, None], zb[:, None])
    got = oracle.window(z, h, w, r, looks, 1.0)
    # d_AB from LAPACK log-determinants (independent of the oracle)
    fa, fb = oracle.to_full(za[:, None])[0], oracle.to_full(zb[:, None])[0]
    dab = looks * (np.linalg.slogdet((fa + fb) / 2)[1]
                   - 0.5 * (np.linalg.slogdet(fa)[1] + np.linalg.slogdet(fb)[1]))
    for p in range(h * w):
        y, x = divmod(p, w)
        ys = range(max(0, y - r), min(h, y + r + 1))
        xr = range(max(0, x - r), min(w, x + r + 1))
        same = sum(1 for _ in ys for xx in xr if (xx < 5) == (x < 5))
        other = len(ys) * len(xr) - same
        assert got[p] == pytest.approx(same + other * math.exp(-dab), rel=1e-13)


def test_pair_distance_properties():
    z = rand_kappa(200, 16, 1e3)
    for p in range(0, 200, 2):
        zi, zj = z[:, p], z[:, p + 1]
        assert oracle.pair_distance(zi, zi, 4.0) == 0.0
        dij = oracle.pair_distance(zi, zj, 4.0)
        assert dij == pytest.approx(oracle.pair_distance(zj, zi, 4.0), rel=1e-15, abs=1e-18)
        assert dij >= 0.0  # log-det concavity
        # det is homogeneous: d_ij(k Z_i, k Z_j) = d_ij
        assert oracle.pair_distance(3.7 * zi, 3.7 * zj, 4.0) == pytest.approx(dij, rel=1e-12, abs=1e-15)


def test_window_brute_force_tiny():
    h, w, r, looks, hh = 5, 6, 2, 4.0, 1.0
    z = rand_kappa(h * w, 17, 50.0)
    got = oracle.window(z, h, w, r, looks, hh)
    full = oracle.to_full(z)
    ld = np.log(np.linalg.det(full).real)
    for p in range(h * w):
        y, x = divmod(p, w)
        acc = 0.0
        for yy in range(max(0, y - r), min(h, y + r + 1)):
            for xx in range(max(0, x - r), min(w, x + r + 1)):
                q = yy * w + xx
                ds = np.log(np.linalg.det((full[p] + full[q]) / 2).real)
                acc += math.exp(-looks * (ds - 0.5 * (ld[p] + ld[q])) / hh)
        assert got[p] == pytest.approx(acc, rel=1e-12)


def test_window_power_form_equivalence():
    # h = 1, L = 4: exp(-d_ij) = ((D_i/D_S)(D_j/D_S))^2 with D_S = det((Z_i+Z_j)/2)
    # (the form the CUDA kernel may use) -- checked on the oracle's own d_ij.
    z = rand_kappa(40, 18, 100.0)
    full = oracle.to_full(z)
    for p in range(0, 40, 2):
        dij = oracle.pair_distance(z[:, p], z[:, p + 1], 4.0)
        di, dj = np.linalg.det(full[p]).real, np.linalg.det(full[p + 1]).real
        ds = np.linalg.det((full[p] + full[p + 1]) / 2).real
        assert math.exp(-dij) == pytest.approx(((di / ds) * (dj / ds)) ** 2, rel=1e-12)


# ------------------------------------------------- multi-frequency blocks (§V)

def _block_full(z, nb):
    n = z.shape[1]
    full = np.zeros((n, 3 * nb, 3 * nb), dtype=np.complex128)
    for b in range(nb):
        full[:, 3 * b:3 * b + 3, 3 * b:3 * b + 3] = oracle.to_full(z[9 * b:9 * b + 9])
    return full


@pytest.mark.parametrize("nb", [1, 2, 3, 4])
def test_blocks_lapack_full_matrix(nb):
    """The blockwise oracle equals LAPACK on the full 3B x 3B block-diagonal
    matrix: inverse (every block, and zero off-diagonal blocks by
    construction) and determinant."""
    z = np.concatenate([rand_kappa(500, 20 + b, 100.0) for b in range(nb)], axis=0)
    out = oracle.inv_det_blocks(z, nb)
    full = _block_full(z, nb)
    inv = np.linalg.inv(full)
    det = np.linalg.det(full)
    for b in range(nb):
        blk = inv[:, 3 * b:3 * b + 3, 3 * b:3 * b + 3]
        assert np.all(normwise(out[9 * b:9 * b + 9], pack(blk)) <= 1e-13)
        # off-diagonal blocks of the LAPACK inverse vanish
        for c in range(nb):
            if c != b:
                assert np.abs(inv[:, 3 * b:3 * b + 3, 3 * c:3 * c + 3]).max() <= 1e-13 * np.abs(inv).max()
    np.testing.assert_allclose(out[9 * nb], det.real, rtol=1e-13)
    np.testing.assert_allclose(out[9 * nb + 1], 1 / det.real, rtol=1e-13)


def test_blocks_single_block_is_inv_det():
    z = rand_hpd(300, 30)
    a = oracle.inv_det_blocks(z, 1)
    b = oracle.inv_det(z)
    assert np.array_equal(a, b)


# ---------------------------------------------------------------- NLM oracle

def test_nlm_constant_image():
    h, w, r = 7, 9, 3
    z0 = rand_hpd(1, 40)[:, 0]
    z = np.repeat(z0[:, None], h * w, axis=1)
    zhat, W = oracle.nlm(z, h, w, r, 4.0, 1.0)
    np.testing.assert_allclose(zhat, z, rtol=1e-15, atol=1e-15 * np.abs(z0).max())
    ref = np.array([clipped_count(p // w, p % w, h, w, r) for p in range(h * w)], float)
    assert np.array_equal(W, ref)


def test_nlm_two_class_closed_form():
    h, w, r, looks = 6, 10, 2, 4.0
    za, zb = rand_hpd(2, 41)[:, 0], rand_hpd(2, 41)[:, 1]
    xs = np.arange(h * w) % w
    z = np.where(xs[None, :] < 5, za[:, None], zb[:, None])
    zhat, W = oracle.nlm(z, h, w, r, looks, 1.0)
    fa, fb = oracle.to_full(za[:, None])[0], oracle.to_full(zb[:, None])[0]
    dab = looks * (np.linalg.slogdet((fa + fb) / 2)[1]
                   - 0.5 * (np.linalg.slogdet(fa)[1] + np.linalg.slogdet(fb)[1]))
    e = math.exp(-dab)
    for p in range(h * w):
        y, x = divmod(p, w)
        ys = range(max(0, y - r), min(h, y + r + 1))
        xr = range(max(0, x - r), min(w, x + r + 1))
        same = sum(1 for _ in ys for xx in xr if (xx < 5) == (x < 5))
        other = len(ys) * len(xr) - same
        zs, zo = (za, zb) if x < 5 else (zb, za)
        ref = (same * zs + other * e * zo) / (same + other * e)
        np.testing.assert_allclose(zhat[:, p], ref, rtol=1e-12, atol=1e-13)
        assert W[p] == pytest.approx(same + other * e, rel=1e-13)


def test_nlm_brute_force_tiny():
    h, w, r, looks, hh = 4, 5, 1, 4.0, 1.0
    z = rand_kappa(h * w, 42, 30.0)
    zhat, W = oracle.nlm(z, h, w, r, looks, hh)
    full = oracle.to_full(z)
    ld = np.log(np.linalg.det(full).real)
    for p in range(h * w):
        y, x = divmod(p, w)
        num = np.zeros(9)
        den = 0.0
        for yy in range(max(0, y - r), min(h, y + r + 1)):
            for xx in range(max(0, x - r), min(w, x + r + 1)):
                q = yy * w + xx
                ds = np.log(np.linalg.det((full[p] + full[q]) / 2).real)
                wq = math.exp(-looks * (ds - 0.5 * (ld[p] + ld[q])) / hh)
                num += wq * z[:, q]
                den += wq
        np.testing.assert_allclose(zhat[:, p], num / den, rtol=1e-11, atol=1e-12)
        assert W[p] == pytest.approx(den, rel=1e-12)


# ------------------------------------------------------------- KL window oracle

def test_kl_distance_properties():
    z = rand_kappa(100, 50, 1e3)
    for p in range(0, 100, 2):
        zi, zj = z[:, p], z[:, p + 1]
        # d_ii = 0 up to the long-double inverse error (~ kappa^2 2^-64, kappa <= 1e3)
        assert abs(oracle.kl_distance(zi, zi, 4.0)) <= 1e-12
        d = oracle.kl_distance(zi, zj, 4.0)
        assert d >= 0  # KL divergence
        assert d == pytest.approx(oracle.kl_distance(zj, zi, 4.0), rel=1e-15)
        # LAPACK special case
        fi, fj = oracle.to_full(zi[:, None])[0], oracle.to_full(zj[:, None])[0]
        ref = 4.0 * ((np.trace(np.linalg.inv(fi) @ fj) + np.trace(np.linalg.inv(fj) @ fi)).real / 2 - 3)
        assert d == pytest.approx(ref, rel=1e-9, abs=1e-12)
        # invariant under congruence Z -> A Z A^H (KL between Wisharts is)
        a = np.array([[2, 1j, 0], [0, 1, 0.5], [0.3, 0, 1]])
        ci = pack((a @ fi @ np.conj(a.T))[None])[:, 0]
        cj = pack((a @ fj @ np.conj(a.T))[None])[:, 0]
        assert oracle.kl_distance(ci, cj, 4.0) == pytest.approx(d, rel=1e-7, abs=1e-10)


def test_window_kl_constant_and_two_class():
    h, w, r = 6, 10, 2
    za, zb = rand_hpd(2, 51)[:, 0], rand_hpd(2, 51)[:, 1]
    zc = np.repeat(za[:, None], h * w, axis=1)
    got = oracle.window_kl(zc, h, w, r, 4.0, 1.0)
    ref = np.array([clipped_count(p // w, p % w, h, w, r) for p in range(h * w)], float)
    np.testing.assert_allclose(got, ref, rtol=1e-15)
    xs = np.arange(h * w) % w
    z = np.where(xs[None, :] < 5, za[:, None], zb[:, None])
    got = oracle.window_kl(z, h, w, r, 4.0, 1.0)
    fa, fb = oracle.to_full(za[:, None])[0], oracle.to_full(zb[:, None])[0]
    dab = 4.0 * ((np.trace(np.linalg.inv(fa) @ fb) + np.trace(np.linalg.inv(fb) @ fa)).real / 2 - 3)
    for p in range(h * w):
        y, x = divmod(p, w)
        ys = range(max(0, y - r), min(h, y + r + 1))
        xr = range(max(0, x - r), min(w, x + r + 1))
        same = sum(1 for _ in ys for xx in xr if (xx < 5) == (x < 5))
        other = len(ys) * len(xr) - same
        assert got[p] == pytest.approx(same + other * math.exp(-dab), rel=1e-12)


# ---------------------------------------------------------------------------
# The float32 entry points.  Every oracle function has a float32 loader of its
# own (oracle/polsar_oracle.c: load_*_f32, the *_f32 wrappers and the is32
# branch of window_kl_any).  fp32 -> binary128 / long double is exact, so a
# float32 call must equal the float64 call on the exactly upcast inputs BIT
# FOR BIT; the float64 entry points are pinned above.  A wrong plane index or
# stride in a float32 loader fails here.  (PAPER.md:168-189, 390-409 [Eq. 3-5];
# BASELINE configs[4] for the window; PAPER.md:1043-1055 [§V] for blocks.)
# ---------------------------------------------------------------------------
def _bits_equal(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_f32_inv_det_equals_f64_on_upcast():
    z32 = rand_kappa(4000, 71, 1e3).astype(np.float32)
    z32[:, :50] = rand_hpd(50, 72, scale_spread=True).astype(np.float32)
    o32, im32 = oracle.inv_det(z32, with_imag=True)
    o64, im64 = oracle.inv_det(z32.astype(np.float64), with_imag=True)
    assert _bits_equal(o32, o64) and _bits_equal(im32, im64)


@pytest.mark.parametrize("nb", [1, 2, 3])
def test_f32_blocks_equals_f64_on_upcast(nb):
    z32 = np.concatenate([rand_hpd(700, 80 + b).astype(np.float32) for b in range(nb)])
    assert _bits_equal(oracle.inv_det_blocks(z32, nb),
                       oracle.inv_det_blocks(z32.astype(np.float64), nb))


def _window_case():
    h, w, r = 9, 13, 3
    z32 = rand_hpd(h * w, 91).astype(np.float32)
    idx = np.array([0, 5, 12, 13, 40, 58, 77, h * w - 1], dtype=np.int64)
    return z32, h, w, r, idx


def test_f32_window_equals_f64_on_upcast():
    z32, h, w, r, idx = _window_case()
    for looks, hh in ((4.0, 1.0), (3.0, 0.7)):
        assert _bits_equal(oracle.window(z32, h, w, r, looks, hh, idx),
                           oracle.window(z32.astype(np.float64), h, w, r, looks, hh, idx))


def test_f32_window_kl_equals_f64_on_upcast():
    z32, h, w, r, idx = _window_case()
    assert _bits_equal(oracle.window_kl(z32, h, w, r, 4.0, 1.0, idx),
                       oracle.window_kl(z32.astype(np.float64), h, w, r, 4.0, 1.0, idx))


def test_f32_nlm_equals_f64_on_upcast():
    z32, h, w, r, idx = _window_case()
    zh32, w32 = oracle.nlm(z32, h, w, r, 4.0, 1.0, idx)
    zh64, w64 = oracle.nlm(z32.astype(np.float64), h, w, r, 4.0, 1.0, idx)
    assert _bits_equal(zh32, zh64) and _bits_equal(w32, w64)


# ---------------------------------------------------------------------------
# The storage-precision instantiation (oracle_inv_det_plain_s / _d, SURVEY
# §8(d)'s plain CPU baseline; timed by bench.py, built -O3 -march=native).
# Pinned to the worked examples (exact for the dyadic ones) and to the
# binary128 definition within the rounding error of the cofactor expansion,
# which grows like kappa^2 u (R-16): a dropped term, wrong sign or
# transposed operand gives O(1) errors and fails.
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("row", parse_golden(), ids=lambda r: r[0])
def test_plain_worked_examples(dt, row):
    name, zin, inv, det, idet = row
    out = oracle.inv_det_plain(zin.reshape(9, 1).astype(dt), 1)
    assert out.dtype == dt
    u = np.finfo(dt).eps
    if name in ("identity", "diag245", "golden"):
        assert np.array_equal(out[:9, 0], inv.astype(dt))
        assert out[9, 0] == det and out[10, 0] == dt(idet)
    else:
        np.testing.assert_allclose(out[:9, 0], inv, rtol=0, atol=8 * u * np.abs(inv).max())
        assert out[9, 0] == pytest.approx(det, rel=8 * u)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("threads", [1, 3])
def test_plain_against_binary128(dt, threads):
    z = np.concatenate([rand_hpd(3000, 11), rand_kappa(3000, 12, 1e2)], axis=1).astype(dt)
    ref = oracle.inv_det(z)
    got = oracle.inv_det_plain(z, threads).astype(np.float64)
    k = oracle.kappa2(z)
    u = float(np.finfo(dt).eps) / 2
    inv = normwise(got[:9], ref[:9])
    det = np.abs(got[9] - ref[9]) / np.abs(ref[9])
    idet = np.abs(got[10] - ref[10]) / np.abs(ref[10])
    bound = 32 * k ** 2 * u
    assert np.all(inv <= bound) and np.all(det <= bound) and np.all(idet <= bound + 2 * u)
    # and it is the storage-precision evaluation, not a wider one
    assert inv.max() > u / 4
