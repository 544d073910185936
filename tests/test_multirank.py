"""The N > 1 host path on CPU: world_size-2 gloo runs of the z-slab protocol
(paper_2501_04229_b200/partition.py) — halo exchange + rank-ordered pairwise
reductions — checked bit for bit against the single-process oracle."""
import os
import socket

import numpy as np
import pytest

from paper_2501_04229_b200.partition import pairwise_tree, slab_plan


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_slab_plan():
    s0, s1 = slab_plan(8, 2, 0), slab_plan(8, 2, 1)
    assert (s0.plane_lo, s0.plane_hi, s0.halo_lo, s0.halo_hi) == (0, 4, False, True)
    assert (s1.plane_lo, s1.plane_hi, s1.halo_lo, s1.halo_hi) == (4, 8, True, False)
    assert s1.row_lo == 256 and s1.rows == 256
    with pytest.raises(ValueError):
        slab_plan(6, 4, 0)


def test_pairwise_tree_matches_oracle(orc):
    rng = np.random.default_rng(0)
    x = orc.round(rng.uniform(-1, 1, 1024), 1)
    y = orc.round(rng.uniform(-1, 1, 1024), 1)
    parts = [orc.dot(x[i * 256:(i + 1) * 256], y[i * 256:(i + 1) * 256], 1) for i in range(4)]
    tot = pairwise_tree(parts, lambda a, b: orc.round(a + b, 1))
    assert tot == orc.dot(x, y, 1)


def _stencil_rows_double(n, t, x_planes, plane_lo, planes):
    """b - A x fold (kernels.cpp:63-66) for the owned planes, binary64, with
    x_planes[q] the (n*n,) plane q of x (halos included)."""
    out = np.empty(planes * n * n)
    nn = n * n
    for pi in range(planes):
        i = plane_lo + pi
        for j in range(n):
            for k in range(n):
                acc = 0.0
                if i > 0:
                    acc = acc + t[0] * x_planes[i - 1][j * n + k]
                if j > 0:
                    acc = acc + t[1] * x_planes[i][(j - 1) * n + k]
                if k > 0:
                    acc = acc + t[2] * x_planes[i][j * n + k - 1]
                acc = acc + t[3] * x_planes[i][j * n + k]
                if k + 1 < n:
                    acc = acc + t[4] * x_planes[i][j * n + k + 1]
                if j + 1 < n:
                    acc = acc + t[5] * x_planes[i][(j + 1) * n + k]
                if i + 1 < n:
                    acc = acc + t[6] * x_planes[i + 1][j * n + k]
                out[pi * nn + j * n + k] = acc
    return out


def _worker(rank, world, port, n, q):
    import torch
    import torch.distributed as dist

    from oracle import Oracle
    from paper_2501_04229_b200.partition import allreduce_pairwise, exchange_halos, slab_plan

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        orc = Oracle()
        N = n ** 3
        A = orc.convdiff(n)
        x, _ = orc.make_rhs(A, 3, -1.0, 1.0)
        slab = slab_plan(n, world, rank)
        lo, hi = slab.row_lo, slab.row_lo + slab.rows
        # 1. pairwise dot in binary16 / binary32 / binary64 over slabs == global
        res = {}
        for p in (0, 1, 2):
            xr = orc.round(x, p)
            part = orc.dot(xr[lo:hi], xr[lo:hi], p)
            res[f"dot{p}"] = allreduce_pairwise(part, lambda a, b, p=p: orc.round(a + b, p))
        # 2. halo exchange + local stencil rows == global matvec rows
        nn = n * n
        planes = {pl: x[pl * nn:(pl + 1) * nn] for pl in range(slab.plane_lo, slab.plane_hi)}
        below, above = exchange_halos(slab, torch.from_numpy(planes[slab.plane_lo].copy()),
                                      torch.from_numpy(planes[slab.plane_hi - 1].copy()))
        if below is not None:
            planes[slab.plane_lo - 1] = below.numpy()
        if above is not None:
            planes[slab.plane_hi] = above.numpy()
        r = 1.0 / (2.0 * n + 2.0)  # problems.hpp:16-22
        t = [-1.0 - r, -1.0 - r, -1.0 - r, 6.0, -1.0 + r, -1.0 + r, -1.0 + r]
        local = _stencil_rows_double(n, t, planes, slab.plane_lo, slab.planes)
        full = orc.matvec(A, x, 2)
        res["matvec_ok"] = bool(np.array_equal(local.view(np.int64), full[lo:hi].view(np.int64)))
        # 3. the bench's max-over-ranks timing
        tt = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        res["max"] = tt.item()
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_slab_protocol(orc, world):
    import torch.multiprocessing as mp

    n = 8
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    A = orc.convdiff(n)
    x, _ = orc.make_rhs(A, 3, -1.0, 1.0)
    for p in (0, 1, 2):
        want = orc.dot(orc.round(x, p), orc.round(x, p), p)
        for r in range(world):
            got = out[r][f"dot{p}"]
            assert np.array([got]).view(np.int64)[0] == np.array([want]).view(np.int64)[0], (p, r, got, want)
    for r in range(world):
        assert out[r]["matvec_ok"]
        assert out[r]["max"] == float(world)
