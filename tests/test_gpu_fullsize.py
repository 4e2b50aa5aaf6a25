"""Parity at BASELINE's full sizes (configs[2] c3, configs[3] c4: 10000 x 40000
pixels), in the launch configuration bench.py times (polsar_inv_det over the
whole image with the status plane, inputs resident in HBM).

The oracle cannot redo 4e8 matrices, so: (1) sampled pixels -- their inputs
regenerated on the host by the generator's bit-identical twin (and compared
bit for bit with the GPU's copy), their outputs computed by the oracle; and
(2) properties checked on every pixel with torch reductions on the device.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_1807_08084_b200 as P
from paper_1807_08084_b200 import configs, wishart
from tests._metrics import TOL, errors, status_expected

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def sample_pixels(n, width, seed, k=20000):
    rng = np.random.default_rng(seed)
    special = [0, 1, 2, 3, width - 1, width, n // 2, n - 5, n - 4, n - 3, n - 2, n - 1]
    return np.unique(np.concatenate([special, rng.integers(0, n, k)])).astype(np.int64)


def check_sampled(cfg, tab, z, out, status, idx, tol):
    zs_host = wishart.generate_pixels_cpu(cfg, idx, table=tab)
    ii = torch.as_tensor(idx, device=z.device)
    zs_gpu = z[:, ii].cpu().numpy()
    assert np.array_equal(zs_host.view(np.uint8), zs_gpu.view(np.uint8))
    ref = oracle.inv_det(zs_host)
    got = out[:, ii].cpu().numpy().astype(np.float64)
    st = status[ii].cpu().numpy()
    k = oracle.kappa2(zs_host)
    m = k <= 1e4
    inv, det, idet = errors(got, ref)
    worst = max(inv[m].max(), det[m].max(), idet[m].max())
    assert worst <= tol, worst
    exp, dec = status_expected(zs_host, ref, cfg.dtype)
    assert np.array_equal(st[dec], exp[dec])
    print(f"\n[report] {cfg.name}: sampled {idx.size} px, kappa<=1e4: {int(m.sum())}, "
          f"max rel err {worst:.2e}, flagged SINGULAR {int((st != 0).sum())} "
          f"(of which kappa<=1e4: {int((st[m] != 0).sum())})")
    return k, inv, det


def full_properties(out, status, dt, algo="adjugate"):
    """Every pixel: OK pixels are finite with det > 0 and det * t within
    rounding of 1 (Alg. 2: t = RN(1/det), a few u; Alg. 1: det and det^-1
    are separate products of rounded factors (R-14), ~6 roundings each)."""
    ok = status == 0
    n_ok = int(ok.sum())
    assert n_ok > 0.98 * status.numel()
    for k in range(11):
        assert bool(torch.isfinite(out[k][ok]).all())
    det = out[9][ok].double()
    t = out[10][ok].double()
    assert bool((det > 0).all())
    u = 2.0 ** -24 if dt == torch.float32 else 2.0 ** -53
    assert float((det * t - 1).abs().max()) <= (4 if algo == "adjugate" else 16) * u


@pytest.fixture(scope="module")
def c3(cuda):
    cfg = configs.get("c3")
    tab = cfg.table()
    z = wishart.generate(cfg, device=cuda, table=tab)
    yield cfg, tab, z
    del z
    torch.cuda.empty_cache()


@pytest.mark.parametrize("algo", ["adjugate", "cholesky"])
def test_c3_full_size(c3, algo):
    cfg, tab, z = c3
    n = z.shape[1]
    out = torch.empty((11, n), dtype=z.dtype, device=z.device)
    status = torch.empty(n, dtype=torch.uint8, device=z.device)
    fn = P.polsar_inv_det if algo == "adjugate" else P.polsar_inv_det_cholesky
    fn(z, out, status)
    torch.cuda.synchronize()
    idx = sample_pixels(n, cfg.width, seed=3)
    check_sampled(cfg, tab, z, out, status, idx, TOL["float32"])
    full_properties(out, status, torch.float32, algo)
    del out, status


@pytest.mark.parametrize("algo", ["adjugate", "cholesky", "adjugate_eft"])
def test_c4_full_size(cuda, algo):
    cfg = configs.get("c4")
    tab = cfg.table()
    z = wishart.generate(cfg, device=cuda, table=tab)
    n = z.shape[1]
    out = torch.empty((11, n), dtype=z.dtype, device=z.device)
    status = torch.empty(n, dtype=torch.uint8, device=z.device)
    if algo == "cholesky":
        P.polsar_inv_det_cholesky(z, out, status)
    else:
        P.polsar_inv_det(z, out, status, eft=algo == "adjugate_eft")
    torch.cuda.synchronize()
    idx = sample_pixels(n, cfg.width, seed=4, k=30000)
    # POLSAR_F64_EFT holds a few ulp (R-16); the others BASELINE's 1e-12
    tol = 2e-15 if algo == "adjugate_eft" else TOL["float64"]
    k, inv, det = check_sampled(cfg, tab, z, out, status, idx, tol)
    # the 1 % near-singular pixels (kappa = 1e6) are reported, not asserted;
    # the error-free Alg. 2 still lands near u * kappa there
    near = k > 1e5
    assert near.sum() > 100
    print(f"\n[report] c4 near-singular pixels: {int(near.sum())} sampled, "
          f"max normwise inverse error {inv[near].max():.2e}, det {det[near].max():.2e}")
    full_properties(out, status, torch.float64, "cholesky" if algo == "cholesky" else "adjugate")
    del out, status, z
    torch.cuda.empty_cache()
