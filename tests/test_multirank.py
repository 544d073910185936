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


# ------------------------------------------------------------ CSR row blocks
def test_row_block_plan():
    from paper_2501_04229_b200.partition import row_block_plan

    b = row_block_plan(1 << 12, 4, 1, 300)
    assert (b.row_lo, b.row_hi, b.win_lo, b.win_hi) == (1024, 2048, 724, 2348)
    assert row_block_plan(1 << 12, 4, 0, 300).win_lo == 0
    assert row_block_plan(1 << 12, 4, 3, 300).win_hi == 1 << 12
    with pytest.raises(ValueError):
        row_block_plan(1000, 3, 0, 10)   # world not a power of two
    with pytest.raises(ValueError):
        row_block_plan(1002, 4, 0, 10)   # world does not divide N
    with pytest.raises(ValueError):
        row_block_plan(1024, 4, 0, 300)  # band wider than a block


def _rb_worker(rank, world, port, N, band, q):
    import torch
    import torch.distributed as dist

    from oracle import CSR, Oracle
    from paper_2501_04229_b200.partition import allreduce_pairwise, exchange_band, row_block_plan, window_csr

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        orc = Oracle()
        A = orc.band(N, 8, band, 7)
        x, _ = orc.make_rhs(A, 5, -1.0, 1.0)
        blk = row_block_plan(N, world, rank, band)
        lo, hi = blk.row_lo, blk.row_hi
        res = {}
        # 1. the split of the window, cropped to the block == the global split's block rows
        wrp, wci, wv = window_csr(A.rp, A.ci, A.v, blk.win_lo, blk.win_hi)
        Hw, Sw = orc.regularize(CSR(blk.win_hi - blk.win_lo, wrp, wci, wv), 0.7)
        Hg, Sg = orc.regularize(A, 0.7)
        a, b = lo - blk.win_lo, hi - blk.win_lo
        ok = True
        for Mw, Mg in ((Hw, Hg), (Sw, Sg)):
            sl_w = slice(Mw.rp[a], Mw.rp[b])
            sl_g = slice(Mg.rp[lo], Mg.rp[hi])
            ok &= np.array_equal(Mw.ci[sl_w] + blk.win_lo, Mg.ci[sl_g])
            ok &= np.array_equal(Mw.v[sl_w].view(np.int64), Mg.v[sl_g].view(np.int64))
            ok &= np.array_equal(Mw.rp[a:b + 1] - Mw.rp[a], Mg.rp[lo:hi + 1] - Mg.rp[lo])
        res["split_ok"] = bool(ok)
        # 2. band exchange + the block's rows of A x == the global matvec's rows
        xo = exchange_band(blk, torch.from_numpy(x[lo:hi].copy())).numpy()
        off = max(0, lo - band)
        y = np.empty(hi - lo)
        for i in range(lo, hi):
            acc = 0.0
            for k in range(A.rp[i], A.rp[i + 1]):
                acc = acc + A.v[k] * xo[A.ci[k] - off]
            y[i - lo] = acc
        res["matvec_ok"] = bool(np.array_equal(y.view(np.int64), orc.matvec(A, x, 2)[lo:hi].view(np.int64)))
        # 3. block partials folded in rank order == the global pairwise dot
        res["dot"] = allreduce_pairwise(orc.dot(x[lo:hi], x[lo:hi], 1), lambda u, v: orc.round(u + v, 1))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_gloo_row_block_protocol(orc):
    import torch.multiprocessing as mp

    world, N, band = 2, 512, 60
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_rb_worker, args=(r, world, port, N, band, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    A = orc.band(N, 8, band, 7)
    x, _ = orc.make_rhs(A, 5, -1.0, 1.0)
    want = orc.dot(x, x, 1)
    for r in range(world):
        assert out[r]["split_ok"] and out[r]["matvec_ok"]
        assert np.array([out[r]["dot"]]).view(np.int64)[0] == np.array([want]).view(np.int64)[0]


# ------------------------------------------------------------ GPR query shards
def test_query_shard_covers_all():
    from paper_2501_04229_b200.partition import query_shard

    for q_len in (0, 1, 5, 64, 65536, 65537):
        for world in (1, 2, 3, 8):
            spans = [query_shard(q_len, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == q_len
            assert all(spans[r][1] == spans[r + 1][0] for r in range(world - 1))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1


def _qs_worker(rank, world, port, q_len, out_q):
    import torch.distributed as dist

    from paper_2501_04229_b200.partition import gather_queries, query_shard

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        xs = np.arange(q_len, dtype=np.float64) * 0.37 + 1.0
        lo, hi = query_shard(q_len, world, rank)
        # a stand-in for predict(): any per-query function (the queries are independent)
        mean, sd = gather_queries(np.sin(xs[lo:hi]), np.sqrt(xs[lo:hi]), q_len)
        out_q.put((rank, bool(np.array_equal(mean, np.sin(xs)) and np.array_equal(sd, np.sqrt(xs)))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("q_len", [7, 1000])
def test_gloo_query_shards(q_len):
    import torch.multiprocessing as mp

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_qs_worker, args=(r, world, port, q_len, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(out[r] for r in range(world))
