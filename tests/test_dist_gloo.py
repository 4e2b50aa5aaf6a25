"""Multi-process (world_size 2, gloo, CPU) coverage of the N > 1 host path:
row sharding, window halo slabs / exchange, and the scalar reductions."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1807_08084_b200 import dist as pdist


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def host_hash(vals, offset):
    """R1's hash of one uint32 plane (tests/_checksum_ref.py, numpy)."""
    from tests._checksum_ref import checksum
    v = np.asarray(vals, dtype=np.uint64).astype(np.uint32).view(np.float32)[None]
    return checksum(v, offset)[0]


def _worker(rank, world, port, fn, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    finally:
        dist.destroy_process_group()


def spawn(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("height", [1, 7, 10000, 2048])
def test_shard_rows_partition(world, height):
    rows = []
    for r in range(world):
        a, b = pdist.shard_rows(height, world, r)
        rows.extend(range(a, b))
    assert rows == list(range(height))


def test_weak_rows():
    assert pdist.weak_rows(10000, 4, 2) == (40000, 20000, 30000)


@pytest.mark.parametrize("r0,r1,H,R", [(0, 10, 10, 3), (0, 5, 20, 11), (5, 9, 20, 2), (15, 20, 20, 11)])
def test_halo_slab(r0, r1, H, R):
    s0, s1, b, e = pdist.halo_slab(r0, r1, H, R)
    assert s0 == max(0, r0 - R) and s1 == min(H, r1 + R)
    assert s0 + b == r0 and s0 + e == r1


IMG_H, IMG_W, RAD = 23, 5, 3


def _image():
    return torch.arange(9 * IMG_H * IMG_W, dtype=torch.float32).reshape(9, IMG_H * IMG_W)


def _halo_job(rank, world):
    img = _image()
    r0, r1 = pdist.shard_rows(IMG_H, world, rank)
    s0, s1, b, e = pdist.halo_slab(r0, r1, IMG_H, RAD)
    slab = torch.full((9, (s1 - s0) * IMG_W), -1.0)
    slab[:, b * IMG_W:e * IMG_W] = img[:, r0 * IMG_W:r1 * IMG_W]  # own rows only
    pdist.exchange_halos(slab, IMG_W, b, e, RAD)
    return torch.equal(slab, img[:, s0 * IMG_W:s1 * IMG_W])


def test_halo_exchange_gloo():
    res = spawn(_halo_job, 2)
    assert all(res.values())


def test_halo_exchange_gloo_3ranks():
    res = spawn(_halo_job, 3)
    assert all(res.values())


def _small_shard_job(rank, world):
    """H = 7 rows over 3 ranks at R = 3: rank 0 owns 2 rows < R.  Every rank
    must refuse (ValueError from the collective check), none may hang."""
    H, W, R = 7, 4, 3
    r0, r1 = pdist.shard_rows(H, world, rank)
    try:
        pdist.check_halo_geometry(r1 - r0, R)
    except ValueError:
        return "refused"
    return "accepted"


def test_halo_exchange_refuses_small_shards():
    res = spawn(_small_shard_job, 3)
    assert set(res.values()) == {"refused"}


def _rows_job(rank, world):
    """The rows a rank generates (host twin of the generator) equal the same
    rows of the 1-GPU image, under both sharding modes of bench.py: strong
    (one configs[2]-law image split) and weak (an N-times taller image whose
    first rows are the 1-GPU image; the per-row Sigma table is prefix-stable)."""
    from paper_1807_08084_b200 import configs, wishart
    cfg = configs.get("c3").scaled(40, 64)
    one = wishart.generate_cpu(cfg, 0, cfg.height, table=cfg.table())
    r0, r1 = pdist.shard_rows(cfg.height, world, rank)
    strong = wishart.generate_cpu(cfg, r0, r1, table=cfg.table())
    ok_strong = np.array_equal(strong, one[:, r0 * cfg.width:r1 * cfg.width])
    H, w0, w1 = pdist.weak_rows(cfg.height, world, rank)
    weak = wishart.generate_cpu(cfg, w0, w1, table=cfg.table(H), height=H)
    ok_weak = rank != 0 or np.array_equal(weak, one)
    return bool(ok_strong and ok_weak)


def test_rank_rows_equal_single_gpu_image():
    res = spawn(_rows_job, 2)
    assert all(res.values())


def _reduce_job(rank, world):
    vals = (np.arange(1000, dtype=np.uint64) * np.uint64(2654435761)) % np.uint64(2**32)
    r0, r1 = pdist.shard_rows(len(vals), world, rank)
    part = host_hash(vals[r0:r1], r0)
    t = torch.tensor([np.int64(np.uint64(part)), r1 - r0, 0, 0], dtype=torch.int64)
    out, tmax = pdist.reduce_results(t, seconds=0.5 + rank)
    return int(np.uint64(np.int64(out[0].item()))), int(out[1].item()), tmax


def test_reduce_results_gloo():
    res = spawn(_reduce_job, 2)
    vals = (np.arange(1000, dtype=np.uint64) * np.uint64(2654435761)) % np.uint64(2**32)
    full = host_hash(vals, 0)
    for rank, (h, cnt, tmax) in res.items():
        assert h == full       # wrapping sums over ranks == single-rank hash
        assert cnt == 1000
        assert tmax == 1.5     # max over ranks
