"""The seeded input generator (host twin; the GPU build is byte-identical,
tests/test_gpu_gen.py): the multilook law Z = (1/L) sum s s^H, s ~ CN(0, Sigma)
(Eq. 2 with reading R-3) checked by its moments, and the
deterministic elementary functions it is built from."""
import math

import numpy as np
import pytest

import oracle
from paper_1807_08084_b200 import configs, wishart
from paper_1807_08084_b200.wishart import sigma as S


def mc(cfg, rows):
    return wishart.generate_cpu(cfg.scaled(rows, 1000)).astype(np.float64)


def test_elementary_functions():
    rng = np.random.default_rng(0)
    for x in rng.uniform(2.0 ** -53, 1.0, 2000):
        assert abs(wishart.cpu_log(x) - math.log(x)) <= 4e-16 * max(1.0, abs(math.log(x)))
    for u in rng.uniform(0, 1, 2000):
        c, s = wishart.cpu_cossin(u)
        assert abs(c - math.cos(2 * math.pi * u)) <= 2e-15 and abs(s - math.sin(2 * math.pi * u)) <= 2e-15
    for x in rng.uniform(-40, 0, 2000):
        assert abs(wishart.cpu_exp2(x) / 2.0 ** x - 1) <= 4e-16


def test_cholesky_tables_reconstruct_sigma():
    for sig in (S.SIGMA_C1[None], S.random_hpd(8, 0, 5), S.per_row(500, 0, 3)):
        tab = S.cholesky_table(sig)
        np.testing.assert_allclose(S.sigma_from_table(tab), sig, rtol=1e-13, atol=1e-13)


def test_per_row_prefix_stable():
    """Row r's Sigma depends only on (seed, stream, r): the table of a taller
    image starts with the shorter image's table (weak-scaling images of N x H
    rows start with the 1-GPU image)."""
    a = S.per_row(2500, 0, 3)
    for m in (1, 1023, 1024, 1025, 2048):
        assert np.array_equal(S.per_row(m, 0, 3), a[:m])
    c3 = configs.get("c3")
    assert np.array_equal(c3.table(20000)[:c3.height], c3.table())


def test_per_row_condition_numbers():
    sig = S.per_row(2000, 0, 3)
    w = np.linalg.eigvalsh(sig)
    kappa = w[:, 2] / w[:, 0]
    assert kappa.max() <= 1e3 * (1 + 1e-9) and kappa.min() >= 1 - 1e-9
    # log-uniform on [1, 1e3]: the median near sqrt(1e3)
    assert 15 < np.median(kappa) < 60


def test_mean_is_sigma():
    cfg = configs.get("c1")
    z = mc(cfg, 100)  # 1e5 samples
    sig = S.SIGMA_C1
    ref = np.array([sig[0, 0].real, sig[0, 1].real, sig[0, 1].imag, sig[0, 2].real, sig[0, 2].imag,
                    sig[1, 1].real, sig[1, 2].real, sig[1, 2].imag, sig[2, 2].real])
    se = z.std(axis=1) / math.sqrt(z.shape[1])
    assert np.all(np.abs(z.mean(axis=1) - ref) <= 5 * se + 1e-12)


@pytest.mark.parametrize("looks", [4, 8])
def test_wishart_det_moment(looks):
    """E[det Z] = det(Sigma) (L-1)(L-2)/L^2 for the complex Wishart (p = 3)."""
    base = configs.get("c1")
    cfg = configs.Config(**{**base.__dict__, "looks": looks})
    z = mc(cfg, 200)
    det = oracle.inv_det(z)[9]
    ref = np.linalg.det(S.SIGMA_C1).real * (looks - 1) * (looks - 2) / looks ** 2
    assert abs(det.mean() - ref) <= 5 * det.std() / math.sqrt(det.size)


def test_wishart_inverse_moment():
    """E[Z^-1] = L/(L-3) Sigma^-1 (L = 8)."""
    base = configs.get("c1")
    cfg = configs.Config(**{**base.__dict__, "looks": 8})
    z = mc(cfg, 200)
    inv = oracle.inv_det(z)[:9]
    si = np.linalg.inv(S.SIGMA_C1) * 8 / 5
    ref = np.array([si[0, 0].real, si[0, 1].real, si[0, 1].imag, si[0, 2].real, si[0, 2].imag,
                    si[1, 1].real, si[1, 2].real, si[1, 2].imag, si[2, 2].real])
    se = inv.std(axis=1) / math.sqrt(inv.shape[1])
    assert np.all(np.abs(inv.mean(axis=1) - ref) <= 6 * se)


def test_paper_sim_law():
    """Mode PAPER_SIM: Z = G G^H with Re/Im(G) ~ U[-1,1]:
    E[Z] = 3 * 2/3 I = 2 I."""
    cfg = configs.get("ctx_sim").scaled(1, 100000)
    z = wishart.generate_cpu(cfg).astype(np.float64)
    m = z.mean(axis=1)
    np.testing.assert_allclose(m[[0, 5, 8]], 2.0, atol=0.02)
    np.testing.assert_allclose(m[[1, 2, 3, 4, 6, 7]], 0.0, atol=0.02)


def test_determinism_and_prefix_stability():
    cfg = configs.get("c2").scaled(40, 50)
    a = wishart.generate_cpu(cfg)
    b = wishart.generate_cpu(cfg)
    assert np.array_equal(a, b)
    part = wishart.generate_cpu(cfg, 10, 20)
    assert np.array_equal(part, a[:, 10 * 50:20 * 50])
    other = wishart.generate_cpu(configs.Config(**{**cfg.__dict__, "seed": 1}))
    assert not np.array_equal(a, other)
