"""Parity of K1 (Alg. 2) and K2 (Alg. 1) against the CPU oracle, through the
C-ABI (via the thin binding), on seeded synthetic inputs.

Tolerance (BASELINE north_star): max relative error <= 1e-12 (fp64 storage)
and <= 2e-5 (fp32 storage) on the inverse (normwise per pixel, R-10), det and
det^-1, over pixels with kappa_2 <= 1e4.  The *_PLAIN modes (Alg. 2 exactly
as printed, in the storage precision) are reported, not asserted.
"""
import os

import numpy as np
import pytest
import torch

import oracle
import paper_1807_08084_b200 as P
from paper_1807_08084_b200 import configs, wishart
from tests._metrics import TOL, entrywise, errors, status_expected, worst

pytestmark = pytest.mark.gpu
THREADS = len(os.sched_getaffinity(0))
ALGOS = ["adjugate", "cholesky"]


def run(z, algo, plain=False):
    out, st = P.inv_det(z, algo=algo, plain=plain)
    torch.cuda.synchronize()
    return out.cpu().numpy(), st.cpu().numpy()


@pytest.fixture(scope="module")
def c1(cuda):
    cfg = configs.get("c1")
    z = wishart.generate(cfg, device=cuda)
    zh = z.cpu().numpy()
    return z, zh, oracle.inv_det(zh), oracle.kappa2(zh)


@pytest.fixture(scope="module")
def c2(cuda):
    cfg = configs.get("c2")
    z = wishart.generate(cfg, device=cuda)
    zh = z.cpu().numpy()
    return z, zh, oracle.inv_det_threaded(zh, THREADS), oracle.kappa2(zh)


@pytest.mark.parametrize("algo", ALGOS)
def test_c1_fp64_parity(c1, algo):
    z, zh, ref, k = c1
    got, st = run(z, algo)
    mask = k <= 1e4
    assert mask.mean() > 0.99
    assert worst(got, ref, mask) <= TOL["float64"]
    exp, dec = status_expected(zh, ref, "float64")
    assert np.array_equal(st[dec], exp[dec])
    assert np.all(st == 0)


def test_c1_fp64_eft_parity(c1):
    """POLSAR_F64_EFT (the error-free Alg. 2, R-16): a few ulp on
    every pixel, whatever kappa -- far inside BASELINE's 1e-12."""
    z, zh, ref, k = c1
    out, st = P.inv_det(z, eft=True)
    got = out.cpu().numpy()
    assert worst(got, ref, np.isfinite(k)) <= 2e-15
    base, _ = P.inv_det(z)
    # the default POLSAR_F64 form and the error-free one agree within the
    # default form's bound
    assert worst(base.cpu().numpy(), got, k <= 1e4) <= TOL["float64"]


def test_eft_refused_where_not_provided(c1):
    z = c1[0]
    with pytest.raises(ValueError):
        P.inv_det(z, algo="cholesky", eft=True)
    with pytest.raises(ValueError):
        P.inv_det(z.float(), eft=True)
    out = torch.empty((11, z.shape[1]), dtype=z.dtype, device=z.device)
    rc = P.lib().polsar_inv_det_cholesky(P._ptr(z), P._ptr(out), None, z.shape[1], z.shape[1],
                                         P.POLSAR_F64_EFT, None)
    assert rc == 3  # POLSAR_ENOTSUP


@pytest.mark.parametrize("algo", ALGOS)
def test_c2_fp32_parity(c2, algo):
    z, zh, ref, k = c2
    got, st = run(z, algo)
    mask = k <= 1e4
    assert worst(got, ref, mask) <= TOL["float32"]
    # fp32 storage with fp64 arithmetic: every complex entry is within a few
    # fp32 roundings of the oracle, not only normwise
    assert entrywise(got, ref)[mask].max() <= 4 * 2.0 ** -24
    exp, dec = status_expected(zh, ref, "float32")
    assert np.array_equal(st[dec], exp[dec])


@pytest.mark.parametrize("algo", ALGOS)
def test_plain_modes_reported(c1, c2, algo, capsys):
    for name, (z, zh, ref, k) in (("c1", c1), ("c2", c2)):
        got, _ = run(z, algo, plain=True)
        mask = k <= 1e4
        e = worst(got, ref, mask)
        with capsys.disabled():
            print(f"\n[report] {algo} PLAIN {name} {z.dtype}: max rel err {e:.3e} (kappa<=1e4)")
        assert np.isfinite(e)


def test_golden_matrix_catches_l21(cuda):
    # PAPER.md:298 prints l21 = (e - l10 conj(l20)) v1; with it c_i = (1-i)/2, e_i = +i.
    z = torch.tensor([2, 1, 1, 0, 0, 3, 0, 1, 1], dtype=torch.float64, device=cuda).reshape(9, 1)
    for algo in ALGOS:
        got, st = run(z, algo)
        ref = np.array([1, -0.5, -0.5, -0.5, 0.5, 1, 0, -1, 2, 2, 0.5])
        np.testing.assert_allclose(got[:, 0], ref, rtol=2e-15, atol=1e-15)
        assert st[0] == 0


@pytest.mark.parametrize("dt", [torch.float32, torch.float64])
@pytest.mark.parametrize("algo", ALGOS)
def test_ragged_and_misaligned_bit_identical(cuda, dt, algo):
    """Scalar tail / misaligned planes give the same bits as the vector body."""
    cfg = configs.get("c2").scaled(8, 1000)
    z = wishart.generate(cfg, device=cuda).to(dt)
    full, st_full = run(z, algo)
    fn = P.polsar_inv_det if algo == "adjugate" else P.polsar_inv_det_cholesky
    fn(z[:, :1], torch.empty((11, z.shape[1]), dtype=dt, device=cuda)[:, :1], None, n=0)  # no-op
    for n in (1, 3, 5, 7, 1023, 4097, 7990):
        for off in (0, 1, 3):
            for pad in (0, 5):
                ld = n + pad
                zc = torch.empty((9, ld), dtype=dt, device=cuda)
                zc[:, :n].copy_(z[:, off:off + n])
                out = torch.full((11, ld), float("nan"), dtype=dt, device=cuda)
                st = torch.full((n,), 255, dtype=torch.uint8, device=cuda)
                fn(zc[:, :n], out[:, :n], st, n=n)
                torch.cuda.synchronize()
                got = out[:, :n].cpu().numpy()
                assert np.array_equal(got.view(np.uint8), full[:, off:off + n].copy().view(np.uint8))
                assert np.array_equal(st.cpu().numpy(), st_full[off:off + n])


@pytest.mark.parametrize("m", [1, -3, 5])
@pytest.mark.parametrize("dt", [torch.float32, torch.float64])
def test_power_of_two_metamorphic_bit_exact(c2, dt, m):
    z = c2[0].to(dt)
    k = 2.0 ** m
    a, _ = run(z, "adjugate")
    b, _ = run(z * k, "adjugate")
    assert np.array_equal(b[:9], a[:9] / np.asarray(k, a.dtype))
    assert np.array_equal(b[9], a[9] * np.asarray(k ** 3, a.dtype))
    assert np.array_equal(b[10], a[10] / np.asarray(k ** 3, a.dtype))


@pytest.mark.parametrize("dt", [torch.float32, torch.float64])
def test_det_times_reciprocal(c2, dt):
    z = c2[0].to(dt)
    got, st = run(z, "adjugate")
    if dt == torch.float64:
        # t = RN(1/det) exactly: |det t - 1| <= u
        prod = got[9] * got[10]
        assert np.all(np.abs(prod - 1) <= 2.0 ** -52)
    else:
        prod = got[9].astype(np.float64) * got[10].astype(np.float64)
        assert np.all(np.abs(prod - 1) <= 2 * 2.0 ** -24)


@pytest.mark.parametrize("looks", [1, 2])
@pytest.mark.parametrize("storage", ["float32", "float64"])
def test_rank_deficient_flagged_singular(cuda, looks, storage):
    # looks < 3: Z has rank <= 2; in floating point det comes out as
    # +-O(u a d f) -- the scaled threshold (R-5) must flag every pixel.  The
    # data are generated in the storage precision (an fp32 rounding of a
    # rank-2 matrix is a full-rank fp64 matrix and is rightly not flagged).
    base = configs.get("c2").scaled(16, 1000)
    cfg = configs.Config(**{**base.__dict__, "looks": looks, "dtype": storage, "name": f"L{looks}"})
    z = wishart.generate(cfg, device=cuda)
    for algo in ALGOS:
        _, st = run(z, algo)
        assert np.all(st != 0), (looks, storage, algo, np.bincount(st))


def test_looks_ge_3_not_flagged(cuda):
    base = configs.get("c2").scaled(16, 1000)
    cfg = configs.Config(**{**base.__dict__, "looks": 3, "name": "L3"})
    z = wishart.generate(cfg, device=cuda)
    _, st = run(z, "adjugate")
    assert np.mean(st == 0) > 0.999


def test_not_pd_and_nonfinite_status(cuda):
    # indefinite, negative diagonal, NaN input
    cols = [[1, 2, 0, 0, 0, 1, 0, 0, 1],      # |b|^2 > a d: indefinite
            [-1, 0, 0, 0, 0, 1, 0, 0, 1],     # a < 0
            [float("nan"), 0, 0, 0, 0, 1, 0, 0, 1],
            [1, 0, 0, 0, 0, 1, 0, 0, 1]]
    z = torch.tensor(cols, dtype=torch.float64, device=cuda).T.contiguous()
    _, st_adj = run(z, "adjugate")
    _, st_chol = run(z, "cholesky")
    assert list(st_adj) == [1, 1, 1, 0]
    assert list(st_chol) == [2, 2, 2, 0]


@pytest.mark.parametrize("algo", ALGOS)
def test_cross_method_agreement(c1, algo):
    z, zh, ref, k = c1
    a, _ = run(z, "adjugate")
    b, _ = run(z, "cholesky")
    mask = k <= 1e6
    inv, det, idet = errors(a, b.astype(np.float64))
    assert inv[mask].max() <= 1e-9 and det[mask].max() <= 1e-10


def test_checksum_split_invariance(c2):
    z = c2[0]
    out, st = P.inv_det(z)
    n = z.shape[1]
    full = P.polsar_checksum(out, n, 11, 0, st)
    parts = torch.zeros(4, dtype=torch.int64, device=z.device)
    for lo, hi in ((0, 1000), (1000, 777777), (777777, n)):
        P.polsar_checksum(out[:, lo:], hi - lo, 11, lo, st[lo:], result=parts)
    torch.cuda.synchronize()
    assert torch.equal(full, parts)
    assert int(full[1]) == n


def _u64(t):
    return int(np.int64(t).view(np.uint64))


@pytest.mark.parametrize("algo", ALGOS)
def test_checksum_matches_numpy(c2, algo):
    """R1 against an independent numpy evaluation of the hash definition
    (tests/_checksum_ref.py) and a bincount of the status plane, bit-exact,
    on the whole c2 output and on a pixel-offset slice."""
    from tests._checksum_ref import checksum
    z = c2[0]
    out, st = P.inv_det(z, algo=algo)
    n = z.shape[1]
    res = P.polsar_checksum(out, n, 11, 0, st)
    torch.cuda.synchronize()
    oh, sh = out.cpu().numpy(), st.cpu().numpy()
    h, counts = checksum(oh, 0, sh)
    got = res.cpu().numpy()
    assert _u64(got[0]) == h
    assert [int(x) for x in got[1:]] == counts
    lo, hi = 123457, 654321
    res2 = P.polsar_checksum(out[:, lo:], hi - lo, 11, lo, st[lo:])
    torch.cuda.synchronize()
    h2, c2s = checksum(oh[:, lo:hi], lo, sh[lo:hi])
    got2 = res2.cpu().numpy()
    assert _u64(got2[0]) == h2 and [int(x) for x in got2[1:]] == c2s
    # input planes too (9 planes, float32 bit patterns)
    res3 = P.polsar_checksum(z, n, 9, 0)
    torch.cuda.synchronize()
    assert _u64(res3.cpu().numpy()[0]) == checksum(c2[1], 0)[0]


def _host_run(z_host, algo, dt_plain, ws_bytes, status=True):
    n = z_host.shape[1]
    oh = torch.empty((11, z_host.stride(0)), dtype=z_host.dtype).pin_memory()[:, :n]
    sh = torch.empty(n, dtype=torch.uint8).pin_memory() if status else None
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    streams = [torch.cuda.Stream() for _ in range(3)]
    P.polsar_inv_det_host(z_host, oh, sh, ws, streams, algo=algo, plain=dt_plain)
    return oh, sh


@pytest.mark.parametrize("dt", [torch.float32, torch.float64])
@pytest.mark.parametrize("algo", [0, 1])
def test_host_pipeline_matches_device(c2, dt, algo):
    z = c2[0][:, :300_001].to(dt).contiguous()
    n = z.shape[1]
    dev_out, dev_st = P.inv_det(z, algo="adjugate" if algo == 0 else "cholesky")
    zh = z.cpu().pin_memory()
    oh, sh = _host_run(zh, algo, False, 4 << 20)  # small workspace: many chunks
    torch.cuda.synchronize()
    assert torch.equal(oh, dev_out.cpu())
    assert torch.equal(sh, dev_st.cpu())


@pytest.mark.parametrize("algo", [0, 1])
def test_host_pipeline_oracle_c2(c2, algo):
    """f-3 (PAPER.md:947-963 [§IV-C], out-of-core streaming): the chunked
    host path against the ORACLE on all of c2 (fp32 storage), with a chunk
    size that leaves a ragged last chunk (1048576 = 13 x 78592 + 26880)."""
    z, zh, ref, k = c2
    n = zh.shape[1]
    chunk = 78592
    ws_bytes = 3 * (20 * 4 + 1) * chunk
    assert P.polsar_host_chunk_pixels(ws_bytes, P.POLSAR_F32) == chunk and n % chunk
    oh, sh = _host_run(torch.from_numpy(zh).pin_memory(), algo, False, ws_bytes)
    got = oh.numpy().astype(np.float64)
    m = k <= 1e4
    assert worst(got, ref, m) <= TOL["float32"]
    exp, dec = status_expected(zh, ref, "float32")
    assert np.array_equal(sh.numpy()[dec & m], exp[dec & m])


@pytest.mark.parametrize("algo", [0, 1])
def test_host_pipeline_oracle_c4_slice(cuda, algo):
    """The chunked host path on a slice of c4 (fp64 storage, L = 8, 1 % of
    pixels at kappa = 1e6) against the oracle at 1e-12, ragged last chunk,
    and with a strided host view (plane stride > n)."""
    cfg = configs.get("c4")
    n = 250_003
    tab = cfg.table()
    idx = np.arange(n, dtype=np.int64) + 17 * cfg.width   # rows 17.. of the image
    zs = wishart.generate_pixels_cpu(cfg, idx, table=tab)
    ref = oracle.inv_det_threaded(zs, THREADS)
    k = oracle.kappa2(zs)
    m = k <= 1e4
    big = torch.zeros((9, n + 1001), dtype=torch.float64).pin_memory()
    big[:, :n] = torch.from_numpy(zs)
    zh = big[:, :n]
    chunk = 40_000
    ws_bytes = 3 * (20 * 8 + 1) * chunk
    oh, sh = _host_run(zh, algo, False, ws_bytes)
    got = oh.numpy()
    assert worst(got, ref, m) <= TOL["float64"]
    exp, dec = status_expected(zs, ref, "float64")
    assert np.array_equal(sh.numpy()[dec & m], exp[dec & m])
    # and equal to the device path bit for bit
    dev_out, dev_st = P.inv_det(torch.from_numpy(zs).to(cuda), algo="adjugate" if algo == 0 else "cholesky")
    assert torch.equal(oh.contiguous(), dev_out.cpu()) and torch.equal(sh, dev_st.cpu())


def _sparse_host_planes(nplanes, n, ld, dtype):
    """A (nplanes, n) host view with plane stride ld over an anonymous
    MAP_NORESERVE mapping: only the touched pages are ever backed."""
    import mmap
    es = torch.empty(0, dtype=dtype).element_size()
    buf = mmap.mmap(-1, ((nplanes - 1) * ld + n) * es,
                    flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS | 0x4000)  # 0x4000 = MAP_NORESERVE
    return buf, torch.frombuffer(buf, dtype=dtype).as_strided((nplanes, n), (ld, 1))


@pytest.mark.parametrize("algo", [0, 1])
def test_host_pipeline_plane_stride_over_max_pitch(cuda, algo):
    """2D copies cap their pitch at cudaDevAttrMaxPitch (2^31 - 1
    bytes); a UAVSAR-scale fp64 plane stride (4e8 x 8 B) exceeds it.  Here
    ld_host = 2^28 + 64 fp64 elements (2.1 GB pitch, pageable sparse memory):
    the host path must copy plane by plane and still match the oracle."""
    n, ld = 5003, (1 << 28) + 64
    assert ld * 8 > 2 ** 31 - 1
    try:
        bz, zh = _sparse_host_planes(9, n, ld, torch.float64)
        bo, oh = _sparse_host_planes(11, n, ld, torch.float64)
    except (OSError, ValueError, OverflowError) as e:
        pytest.skip(f"cannot map a sparse host buffer: {e}")
    zs = wishart.generate_pixels_cpu(configs.get("c1"), np.arange(n, dtype=np.int64))
    zh.copy_(torch.from_numpy(zs))
    sh = torch.empty(n, dtype=torch.uint8)
    ws = torch.empty(1 << 20, dtype=torch.uint8, device=cuda)   # several chunks
    streams = [torch.cuda.Stream() for _ in range(3)]
    P.polsar_inv_det_host(zh, oh, sh, ws, streams, algo=algo)
    ref = oracle.inv_det(zs)
    assert worst(oh.numpy(), ref, oracle.kappa2(zs) <= 1e4) <= TOL["float64"]
    dev_out, dev_st = P.inv_det(torch.from_numpy(zs).to(cuda), algo="adjugate" if algo == 0 else "cholesky")
    assert torch.equal(oh.clone(), dev_out.cpu()) and torch.equal(sh, dev_st.cpu())


def test_host_pipeline_no_status_and_tiny(cuda):
    """n smaller than one chunk, n = 1, and no status plane."""
    zs = wishart.generate_pixels_cpu(configs.get("c1"), np.arange(7, dtype=np.int64))
    ref = oracle.inv_det(zs)
    for n in (1, 7):
        zh = torch.from_numpy(np.ascontiguousarray(zs[:, :n])).pin_memory()
        oh, _ = _host_run(zh, 0, False, 1 << 20, status=False)
        assert worst(oh.numpy(), ref[:, :n], np.ones(n, bool)) <= TOL["float64"]


@pytest.mark.parametrize("algo", ALGOS)
def test_residual_bound(c1, algo):
    """||M Minv - I||_max <= 64 eps kappa(M) (eps = 2^-53), checked
    with an independent complex matmul on the full Hermitian matrices -- no
    oracle involved."""
    z, zh, ref, k = c1
    out, st = run(z, algo)
    m = oracle.to_full(zh)
    x = oracle.to_full(out[:9])
    r = np.abs(m @ x - np.eye(3)).max(axis=(1, 2))
    ok = (st == 0) & np.isfinite(k)
    ratio = r[ok] / (64 * 2.0 ** -53 * k[ok])
    print(f"[report] {algo} residual / (64 eps kappa): max {ratio.max():.3f}, median {np.median(ratio):.4f}, "
          f"kappa max {k[ok].max():.3g}")
    assert ratio.max() <= 1.0
