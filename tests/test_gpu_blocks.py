"""Multi-frequency block-diagonal pixels (PAPER.md:1043-1055 [§V]; SURVEY
§8(f) row 4): polsar_inv_det_blocks against the blockwise binary128 oracle
(itself pinned to LAPACK on the full 3B x 3B matrix in test_oracle.py)."""
import numpy as np
import pytest
import torch

import oracle
import paper_1807_08084_b200 as P
from paper_1807_08084_b200 import configs, wishart
from tests._metrics import TOL

pytestmark = pytest.mark.gpu


def block_errors(got, ref, nb):
    errs = []
    for b in range(nb):
        g, r = got[9 * b:9 * b + 9], ref[9 * b:9 * b + 9]
        errs.append(np.max(np.abs(g - r), axis=0) / np.max(np.abs(r), axis=0))
    det = np.abs(got[9 * nb] - ref[9 * nb]) / np.abs(ref[9 * nb])
    idet = np.abs(got[9 * nb + 1] - ref[9 * nb + 1]) / np.abs(ref[9 * nb + 1])
    return np.max(np.stack(errs), axis=0), det, idet


@pytest.mark.parametrize("storage", ["float32", "float64"])
@pytest.mark.parametrize("nb", [1, 2, 3])
def test_blocks_parity(cuda, storage, nb):
    base = configs.get("c2").scaled(200, 300)
    cfg = configs.Config(**{**base.__dict__, "dtype": storage})
    z = wishart.generate_bands(cfg, nb, device=cuda)
    zh = z.cpu().numpy()
    assert np.array_equal(zh, wishart.generate_bands_cpu(cfg, nb))
    out = torch.empty((9 * nb + 2, z.shape[1]), dtype=z.dtype, device=cuda)
    st = torch.empty(z.shape[1], dtype=torch.uint8, device=cuda)
    P.polsar_inv_det_blocks(z, out, nb, st)
    torch.cuda.synchronize()
    ref = oracle.inv_det_blocks(zh, nb)
    kmax = np.max(np.stack([oracle.kappa2(zh[9 * b:9 * b + 9]) for b in range(nb)]), axis=0)
    m = kmax <= 1e4
    inv, det, idet = block_errors(out.cpu().numpy().astype(np.float64), ref, nb)
    # BASELINE's bound for every band count: K5 multiplies the block dets in
    # the fp64 arithmetic type (nb - 1 roundings of ~1e-16) and rounds once to
    # the storage type
    worst = max(inv[m].max(), det[m].max(), idet[m].max())
    print(f"[report] blocks {storage} nb={nb}: max rel err {worst:.3e}")
    assert worst <= TOL[storage]
    assert np.all(st.cpu().numpy()[m] == 0)


@pytest.mark.parametrize("dt", [torch.float32, torch.float64])
def test_single_block_equals_inv_det(cuda, dt):
    cfg = configs.get("c2").scaled(20, 999)
    z = wishart.generate(cfg, device=cuda).to(dt)
    a, sa = P.inv_det(z)
    b = torch.empty_like(a)
    sb = torch.empty_like(sa)
    P.polsar_inv_det_blocks(z, b, 1, sb)
    torch.cuda.synchronize()
    assert torch.equal(a, b) and torch.equal(sa, sb)


def test_blocks_status_worst_block(cuda):
    # block 1 rank-deficient (looks = 1) -> the whole pixel is SINGULAR
    base = configs.get("c2").scaled(10, 100)
    good = wishart.generate(base, device=cuda)
    bad = wishart.generate(configs.Config(**{**base.__dict__, "looks": 1, "stream": 77}), device=cuda)
    z = torch.cat([good, bad], dim=0).contiguous()
    out = torch.empty((20, z.shape[1]), dtype=z.dtype, device=cuda)
    st = torch.empty(z.shape[1], dtype=torch.uint8, device=cuda)
    P.polsar_inv_det_blocks(z, out, 2, st)
    torch.cuda.synchronize()
    assert bool((st == 1).all())
