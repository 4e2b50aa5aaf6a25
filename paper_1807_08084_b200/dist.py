"""Multi-GPU plumbing (host side): pixel-row sharding, window halos, and the
scalar reductions.  One process per GPU, torch.distributed for the
collectives (NCCL on B200, gloo in the CPU tests).

The inverse/det path (K1, K2) is embarrassingly parallel over pixels: ranks
own contiguous pixel rows and never exchange data.  The window
path (K3) needs R rows of halo on each side of a rank's rows: either
regenerated locally (the seeded generator is keyed by global pixel, so this is
exact and needs no communication -- the default) or exchanged with the
neighbouring ranks (``exchange_halos``, for inputs that were not generated
in place).  The only collectives on the hot path's result are scalars:
the order-independent output checksum and status counts (SUM) and the kernel
time (MAX), see ``reduce_results``.
"""
from __future__ import annotations


def shard_rows(height: int, world: int, rank: int):
    """Rows [r0, r1) of an image of `height` rows owned by `rank` (strong
    split: floor(r H / P))."""
    if not (0 <= rank < world) or height < 0:
        raise ValueError("bad shard")
    return (rank * height) // world, ((rank + 1) * height) // world


def weak_rows(rows_per_rank: int, world: int, rank: int):
    """Weak scaling: the image has world * rows_per_rank rows, rank r owns a
    fixed-size block.  Returns (image_height, r0, r1)."""
    return rows_per_rank * world, rank * rows_per_rank, (rank + 1) * rows_per_rank


def halo_slab(r0: int, r1: int, height: int, radius: int):
    """In-image slab of rows needed to compute output rows [r0, r1) of a
    (2R+1)^2 window clipped to the image: [max(0, r0-R), min(H, r1+R)).
    Returns (s0, s1, out_begin, out_end) with the output rows relative to s0."""
    s0, s1 = max(0, r0 - radius), min(height, r1 + radius)
    return s0, s1, r0 - s0, r1 - s0


def check_halo_geometry(own_rows: int, radius: int, device=None, group=None):
    """Collective check (all ranks, MIN-reduced) that every rank owns at least
    `radius` rows: then each halo comes from the adjacent rank alone and the
    rows a rank sends equal the rows its neighbour expects.  Raises
    ValueError on every rank otherwise (instead of a mismatched send/recv
    that could hang).  Call once before ``exchange_halos``."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([own_rows], dtype=torch.int64, device=device)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    if int(t.item()) < radius:
        raise ValueError(f"halo exchange needs every rank to own >= R = {radius} rows "
                         f"(smallest shard: {int(t.item())}); use local regeneration")


def exchange_halos(slab, width: int, own_begin: int, own_end: int, radius: int, group=None):
    """Fill the halo rows of `slab` (a (planes, rows*width) tensor holding the
    rank's slab rows, own rows at [own_begin, own_end)) from the neighbouring
    ranks with point-to-point send/recv (NCCL on GPU, gloo on CPU).  Each
    rank sends its first/last `radius` own rows to rank-1 / rank+1.  Slab
    geometry must come from ``halo_slab`` on every rank, and every rank must
    own >= radius rows (``check_halo_geometry``): then a rank's top and bottom
    halos are exactly `radius` rows wherever it has a neighbour, so the rows
    sent and the rows received match on both sides."""
    import torch.distributed as dist

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    ops = []
    top = own_begin                       # halo rows above our own rows
    bot = slab.shape[1] // width - own_end  # halo rows below
    if own_end - own_begin < radius or (rank > 0 and top != radius) or (rank < world - 1 and bot != radius):
        raise ValueError("exchange_halos: every rank must own >= R rows with R-row halos towards "
                         "its neighbours (check_halo_geometry)")
    if rank > 0 and top > 0:
        send = slab[:, own_begin * width:(own_begin + top) * width].contiguous()
        recv = slab[:, :top * width]
        rbuf = recv.contiguous()
        ops.append(dist.P2POp(dist.isend, send, rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, rbuf, rank - 1, group))
        pending_top = (recv, rbuf)
    else:
        pending_top = None
    if rank < world - 1 and bot > 0:
        send = slab[:, (own_end - bot) * width:own_end * width].contiguous()
        recv = slab[:, own_end * width:]
        rbuf = recv.contiguous()
        ops.append(dist.P2POp(dist.isend, send, rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, rbuf, rank + 1, group))
        pending_bot = (recv, rbuf)
    else:
        pending_bot = None
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for p in (pending_top, pending_bot):
        if p is not None and p[0].data_ptr() != p[1].data_ptr():
            p[0].copy_(p[1])
    return slab


def reduce_results(checksum_counts, seconds: float, group=None):
    """SUM the per-rank int64[4] (checksum, status counts) -- int64 addition
    wraps exactly like uint64, so the total equals the single-GPU result bit
    for bit -- and MAX the per-rank kernel seconds.  Returns
    (checksum_counts, max_seconds)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return checksum_counts, seconds
    dist.all_reduce(checksum_counts, op=dist.ReduceOp.SUM, group=group)
    t = torch.tensor([seconds], dtype=torch.float64, device=checksum_counts.device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return checksum_counts, float(t.item())
