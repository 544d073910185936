"""Host-side z-slab partition logic for the multi-GPU solve.

The 3D grid's rows are i*n^2 + j*n + k with i slowest (problems.cpp:14), so
rank r of G owns the contiguous planes [r*n/G, (r+1)*n/G): N/G consecutive
unknowns. One 7-point operator application needs one halo plane from each
neighbour; every dot product / norm needs one scalar exchange.

Determinism and parity: with G and n powers of two each rank's slab is an
aligned power-of-two block of the reference's pairwise-sum tree
(kernels.cpp:33-39), so the G slab partials combined by a perfect binary tree
in rank order give the single-device (and reference) value bit for bit.
`allreduce_pairwise` does exactly that over any torch.distributed backend
(all-gather of the G partials, then the same tree on every rank) instead of
an allreduce whose summation order the backend chooses.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Sequence


@dataclass(frozen=True)
class Slab:
    rank: int
    world: int
    n: int
    plane_lo: int      # first owned plane
    plane_hi: int      # one past the last owned plane
    halo_lo: bool      # needs plane plane_lo-1 from rank-1
    halo_hi: bool      # needs plane plane_hi from rank+1

    @property
    def planes(self) -> int:
        return self.plane_hi - self.plane_lo

    @property
    def row_lo(self) -> int:
        return self.plane_lo * self.n * self.n

    @property
    def rows(self) -> int:
        return self.planes * self.n * self.n


def is_pow2(v: int) -> bool:
    return v > 0 and (v & (v - 1)) == 0


def slab_plan(n: int, world: int, rank: int) -> Slab:
    """Contiguous planes per rank; requires world | n (the bitwise-parity
    guarantee additionally needs n and world powers of two)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if n % world:
        raise ValueError(f"z-slab partition needs world ({world}) to divide n ({n})")
    per = n // world
    lo, hi = rank * per, (rank + 1) * per
    return Slab(rank, world, n, lo, hi, lo > 0, hi < n)


def pairwise_tree(values: Sequence, add: Callable):
    """Perfect binary tree over len(values) (a power of two) in index order."""
    vals = list(values)
    if not is_pow2(len(vals)):
        raise ValueError("pairwise_tree needs a power-of-two count")
    while len(vals) > 1:
        vals = [add(vals[i], vals[i + 1]) for i in range(0, len(vals), 2)]
    return vals[0]


def allreduce_pairwise(partial: float, add: Callable, group=None) -> float:
    """Gather every rank's partial and fold them in rank order on every rank:
    deterministic, identical everywhere, and equal to the single-device
    pairwise sum when the slabs are aligned power-of-two blocks."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    t = torch.tensor([partial], dtype=torch.float64)
    out = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    return pairwise_tree([float(o.item()) for o in out], add)


def exchange_halos(slab: Slab, lo_plane, hi_plane, group=None):
    """Send my first/last owned plane to rank-1/rank+1 and receive theirs.
    lo_plane / hi_plane are contiguous torch tensors (n*n values); returns
    (halo_below, halo_above), None where there is no neighbour."""
    import torch
    import torch.distributed as dist

    reqs = []
    below = above = None
    if slab.halo_lo:
        below = torch.empty_like(lo_plane)
        reqs.append(dist.irecv(below, slab.rank - 1, group=group))
        reqs.append(dist.isend(lo_plane.contiguous(), slab.rank - 1, group=group))
    if slab.halo_hi:
        above = torch.empty_like(hi_plane)
        reqs.append(dist.irecv(above, slab.rank + 1, group=group))
        reqs.append(dist.isend(hi_plane.contiguous(), slab.rank + 1, group=group))
    for r in reqs:
        r.wait()
    return below, above


# ------------------------------------------------------------ CSR row blocks
@dataclass(frozen=True)
class RowBlock:
    """Rank r's contiguous rows [row_lo, row_hi) of an N-row banded CSR
     and the window [win_lo, win_hi) = the block +- the band
    whose rows (restricted to window columns) determine the block's rows of
    H = aI + (A+A^T)/2 and S = aI + (A-A^T)/2 (splitting.cpp:12-20): a row's
    transpose entries come from rows within the band."""
    rank: int
    world: int
    N: int
    band: int
    row_lo: int
    row_hi: int
    win_lo: int
    win_hi: int

    @property
    def rows(self) -> int:
        return self.row_hi - self.row_lo


def row_block_plan(N: int, world: int, rank: int, band: int) -> RowBlock:
    """N / world rows per rank (world a power of two dividing N: every
    rank's block is an aligned node of the pairwise-sum tree); the band may
    not exceed a block (the halo comes from the two neighbours only)."""
    if world < 1 or not 0 <= rank < world or not is_pow2(world):
        raise ValueError("bad rank/world (world: a power of two)")
    if N % world:
        raise ValueError(f"row-block partition needs world ({world}) to divide N ({N})")
    m = N // world
    if band > m:
        raise ValueError(f"band {band} exceeds a row block of {m} rows: use fewer ranks")
    lo, hi = rank * m, (rank + 1) * m
    return RowBlock(rank, world, N, band, lo, hi, max(0, lo - band), min(N, hi + band))


def window_csr(rp, ci, v, lo: int, hi: int):
    """Rows [lo, hi) of a CSR restricted to the columns [lo, hi), columns
    shifted by -lo (what a rank splits; gadi_api.cu create_impl)."""
    import numpy as np

    out_rp, out_ci, out_v = [0], [], []
    for i in range(lo, hi):
        for k in range(rp[i], rp[i + 1]):
            if lo <= ci[k] < hi:
                out_ci.append(ci[k] - lo)
                out_v.append(v[k])
        out_rp.append(len(out_ci))
    return np.array(out_rp, np.int64), np.array(out_ci, np.int64), np.array(out_v, np.float64)


def exchange_band(blk: RowBlock, x_local, group=None):
    """The band of operand entries each SpMV needs beyond the block: my first
    / last `band` entries to rank-1 / rank+1, theirs back. Returns the
    operand over [row_lo - band, row_hi + band) clipped to [0, N)."""
    import torch
    import torch.distributed as dist

    b = blk.band
    reqs = []
    below = above = None
    if blk.rank > 0 and b:
        below = torch.empty(b, dtype=x_local.dtype)
        reqs.append(dist.irecv(below, blk.rank - 1, group=group))
        reqs.append(dist.isend(x_local[:b].contiguous(), blk.rank - 1, group=group))
    if blk.rank + 1 < blk.world and b:
        above = torch.empty(b, dtype=x_local.dtype)
        reqs.append(dist.irecv(above, blk.rank + 1, group=group))
        reqs.append(dist.isend(x_local[-b:].contiguous(), blk.rank + 1, group=group))
    for r in reqs:
        r.wait()
    return torch.cat([t for t in (below, x_local, above) if t is not None])


# ------------------------------------------------------------ GPR query shards
def query_shard(q_len: int, world: int, rank: int):
    """Rank r's contiguous slice [lo, hi) of q_len prediction queries (SURVEY
    §8(e), C5): the queries are independent, so the predictor shards them with
    no data-path exchange; slices differ by at most one query."""
    if not (0 <= rank < world) or q_len < 0:
        raise ValueError("bad shard")
    base, rem = divmod(q_len, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def gather_queries(local_mean, local_sd, q_len: int, group=None):
    """All ranks' slices of (mean, sd) assembled in rank order on every rank
    (one all_gather of padded slices; gloo or nccl)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    width = (q_len + world - 1) // world
    pad = torch.zeros(2, width, dtype=torch.float64)
    pad[0, : len(local_mean)] = torch.as_tensor(np.asarray(local_mean, dtype=np.float64))
    pad[1, : len(local_sd)] = torch.as_tensor(np.asarray(local_sd, dtype=np.float64))
    dev = None
    if dist.get_backend(group) == "nccl":
        dev = torch.device("cuda", torch.cuda.current_device())
        pad = pad.to(dev)
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    mean = np.empty(q_len)
    sd = np.empty(q_len)
    for r in range(world):
        lo, hi = query_shard(q_len, world, r)
        t = parts[r].cpu().numpy()
        mean[lo:hi] = t[0, : hi - lo]
        sd[lo:hi] = t[1, : hi - lo]
    return mean, sd
