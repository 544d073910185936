"""Sharded solves (z-slabs of the stencil, row blocks of a CSR): `world` ranks as threads of one
process sharing the GPU (LocalComm: device copies + host barriers, no kernel
waits on another rank). Each slab is an aligned power-of-two block of every
pairwise-sum tree and the slab partials are folded in rank order, so the
sharded solve returns the single-device solve's x and history bit for bit.
The NCCL transport (one rank per process) runs the same engine code with
ncclAllGather / ncclSend / ncclRecv in place of the device copies."""
import threading

import numpy as np
import pytest
import torch

import paper_2501_04229_b200 as g

pytestmark = pytest.mark.gpu


def bits(t):
    return t.detach().cpu().numpy().view(np.int64)


def run_sharded(S, world, cfg, b, x_out):
    grp = g.ShardGroup.local(world)
    shards = [g.ShardSystem(S, grp, r) for r in range(world)]
    nl = shards[0].n
    assert all(sh.n == nl and sh.first_row == r * nl for r, sh in enumerate(shards))
    ptr = lambda t, r: t.data_ptr() + r * nl * 8
    reps = g.solve_group(shards, cfg, [ptr(b, r) for r in range(world)], [ptr(x_out, r) for r in range(world)])
    for sh in shards:
        sh.close()
    grp.close()
    return reps


@pytest.mark.parametrize("n,world,ur,accum,alpha", [
    (16, 2, g.Precision.Single, g.Accum.Native, 0.3),
    (16, 4, g.Precision.Half, g.Accum.Fp32, 0.4),
    (32, 4, g.Precision.Half, g.Accum.Fp32, 0.4),
    (16, 2, g.Precision.Double, g.Accum.Native, 0.3),
    (32, 8, g.Precision.Single, g.Accum.Native, 0.2),
    (64, 2, g.Precision.Half, g.Accum.Fp32, 0.3),
])
def test_sharded_solve_bitwise(n, world, ur, accum, alpha):
    S = g.build_convdiff3d(n, r=0.3)
    N = S.n_rows
    full = g.CudaGadiSystem(S)
    xt = torch.empty(N, dtype=torch.float64, device="cuda")
    b = torch.empty_like(xt)
    full.make_rhs(1, -1.0, 1.0, xt.data_ptr(), b.data_ptr())
    cfg = g.GadiConfig(alpha=alpha, xi=1e-20, u_r=ur, accum=accum, stall_window=400,
                       inner=g.InnerSolverSpec(g.InnerMethod.Cg, 1e-12, 5, 30))
    x1 = torch.empty_like(xt)
    rep1 = full.solve_device(b.data_ptr(), x1.data_ptr(), cfg)
    full.close()
    xs = torch.full_like(xt, float("nan"))
    reps = run_sharded(S, world, cfg, b, xs)
    torch.cuda.synchronize()
    assert rep1.status == g.SolveStatus.Converged
    for rep in reps:  # every rank took the same decisions
        assert rep.status == rep1.status
        assert rep.outer_iters == rep1.outer_iters
        assert rep.inner_iter_totals == rep1.inner_iter_totals
        assert np.array_equal(rep.rel_residual_history.view(np.int64), rep1.rel_residual_history.view(np.int64))
    assert np.array_equal(bits(xs), bits(x1))


def test_sharded_make_rhs_matches():
    """make_rhs on shards (global-index RNG + a halo of x_true) = the slabs of
    the single-device b, bit for bit; called collectively from one thread per rank."""
    n, world = 32, 4
    S = g.build_convdiff3d(n, r=0.3)
    full = g.CudaGadiSystem(S)
    xt = torch.empty(S.n_rows, dtype=torch.float64, device="cuda")
    b = torch.empty_like(xt)
    full.make_rhs(3, -1.0, 1.0, xt.data_ptr(), b.data_ptr())
    grp = g.ShardGroup.local(world)
    shards = [g.ShardSystem(S, grp, r) for r in range(world)]
    nl = shards[0].n
    xs, bs = torch.empty_like(xt), torch.empty_like(b)
    th = [threading.Thread(target=sh.make_rhs, args=(3, -1.0, 1.0, xs.data_ptr() + r * nl * 8,
                                                      bs.data_ptr() + r * nl * 8)) for r, sh in enumerate(shards)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    assert np.array_equal(bits(xs), bits(xt))
    assert np.array_equal(bits(bs), bits(b))
    for sh in shards:
        sh.close()
    grp.close()


def test_shard_contract_errors():
    S = g.build_convdiff3d(16)
    with pytest.raises(g.ParameterError):
        g.ShardGroup.local(3)
    grp = g.ShardGroup.local(2)
    with pytest.raises(g.GadiError):
        g.ShardSystem(g.build_convdiff3d(15), grp, 0)  # world must divide n
    sh = g.ShardSystem(S, grp, 1)
    assert (sh.first_row, sh.n) == (8 * 256, 8 * 256)
    with pytest.raises(g.GadiError):
        sh.residual_uf(np.zeros(sh.n))  # whole-vector API calls are not collective
    sh.close()
    grp.close()


def test_nccl_transport_world1():
    """The NCCL transport (libnccl loaded at run time, ncclAllGather of the
    reduction records) on a one-rank communicator: the same bits as the
    unsharded solve. Multi-rank NCCL runs under torchrun (bench.py --gpus N)."""
    S = g.build_convdiff3d(16, r=0.3)
    full = g.CudaGadiSystem(S)
    xt = torch.empty(S.n_rows, dtype=torch.float64, device="cuda")
    b = torch.empty_like(xt)
    full.make_rhs(1, -1.0, 1.0, xt.data_ptr(), b.data_ptr())
    cfg = g.GadiConfig(alpha=0.3, xi=1e-20, u_r=g.Precision.Half, accum=g.Accum.Fp32,
                       inner=g.InnerSolverSpec(g.InnerMethod.Cg, 1e-12, 5, 30))
    x1 = torch.empty_like(xt)
    rep1 = full.solve_device(b.data_ptr(), x1.data_ptr(), cfg)
    grp = g.ShardGroup.nccl(1, 0, g.nccl_unique_id())
    sh = g.ShardSystem(S, grp, 0)
    x2 = torch.empty_like(xt)
    rep2 = sh.solve_device(b.data_ptr(), x2.data_ptr(), cfg)
    torch.cuda.synchronize()
    assert rep2.outer_iters == rep1.outer_iters and rep2.status == rep1.status
    assert np.array_equal(bits(x2), bits(x1))
    sh.close()
    grp.close()
    full.close()


# ------------------------------------------------------------ CSR row blocks
# contiguous row blocks of N/world rows; each rank splits
# the window [r0 - band, r1 + band)^2 around its block on its own device, the
# SpMVs exchange the band of operand entries with the neighbours, and the
# block partials of every reduction fold in rank order -- the single-device
# solve bit for bit (world | N, world a power of two).

def _solve_pair(A, world, cfg, seed=1):
    full = g.CudaGadiSystem(A)
    N = A.n_rows
    xt = torch.empty(N, dtype=torch.float64, device="cuda")
    b = torch.empty_like(xt)
    full.make_rhs(seed, -1.0, 1.0, xt.data_ptr(), b.data_ptr())
    x1 = torch.empty_like(xt)
    rep1 = full.solve_device(b.data_ptr(), x1.data_ptr(), cfg)
    full.close()
    xs = torch.full_like(xt, float("nan"))
    reps = run_sharded(A, world, cfg, b, xs)
    torch.cuda.synchronize()
    return rep1, x1, reps, xs


@pytest.mark.parametrize("N,world,band,ur,accum,method", [
    (8192, 2, 300, g.Precision.Half, g.Accum.Fp32, g.InnerMethod.Cg),
    (8192, 4, 300, g.Precision.Single, g.Accum.Native, g.InnerMethod.Cg),
    (16384, 8, 1000, g.Precision.Half, g.Accum.Fp32, g.InnerMethod.Cg),
    (8192, 4, 300, g.Precision.Double, g.Accum.Native, g.InnerMethod.Gmres),
    (4096, 2, 40000, g.Precision.Half, g.Accum.Fp32, g.InnerMethod.Cg),  # band = the block size
])
def test_sharded_band_rows_bitwise(N, world, band, ur, accum, method):
    band = min(band, N // world)
    A = g.build_band_csr(N, 26, band, 3)
    cfg = g.GadiConfig(alpha=3.0, xi=1e-20, u_r=ur, accum=accum, stall_window=400,
                       inner=g.InnerSolverSpec(method, 1e-12, 5, 30))
    rep1, x1, reps, xs = _solve_pair(A, world, cfg)
    assert rep1.status == g.SolveStatus.Converged
    for rep in reps:
        assert rep.status == rep1.status and rep.outer_iters == rep1.outer_iters
        assert rep.inner_iter_totals == rep1.inner_iter_totals
        assert np.array_equal(rep.rel_residual_history.view(np.int64), rep1.rel_residual_history.view(np.int64))
    assert np.array_equal(bits(xs), bits(x1))


def _random_csr(N, band, k, seed):
    """A nonsymmetric, diagonally dominant CSR with ragged rows (0..k
    off-diagonals within +-band), host side (the reference's CSR layout)."""
    rng = np.random.default_rng(seed)
    rp, ci, va = [0], [], []
    for i in range(N):
        cols = rng.integers(max(0, i - band), min(N, i + band + 1), size=rng.integers(0, k + 1))
        cols = np.unique(np.append(cols, i))
        vals = rng.uniform(-1, 1, cols.size)
        vals[cols == i] = 1.2 * np.abs(vals[cols != i]).sum() + 0.5
        ci.extend(cols.tolist()); va.extend(vals.tolist()); rp.append(len(ci))
    return g.SparseMatrix(N, N, np.array(rp), np.array(ci), np.array(va))


@pytest.mark.parametrize("N,world,band", [(3000, 2, 37), (4096, 8, 200), (6000, 4, 1400)])
def test_sharded_csr_rows_bitwise(N, world, band):
    """Host CSR input, ragged rows, non-power-of-two blocks (N/world rows each)."""
    A = _random_csr(N, band, 9, 11)
    cfg = g.GadiConfig(alpha=2.0, xi=1e-20, u_r=g.Precision.Single, stall_window=400,
                       inner=g.InnerSolverSpec(g.InnerMethod.Cg, 1e-12, 5, 30))
    rep1, x1, reps, xs = _solve_pair(A, world, cfg)
    assert rep1.status == g.SolveStatus.Converged
    for rep in reps:
        assert rep.outer_iters == rep1.outer_iters
        assert np.array_equal(rep.rel_residual_history.view(np.int64), rep1.rel_residual_history.view(np.int64))
    assert np.array_equal(bits(xs), bits(x1))


def test_sharded_band_contract():
    """world must divide N; a band wider than a block needs fewer ranks (an
    error, never a silent fallback)."""
    grp = g.ShardGroup.local(4)
    with pytest.raises(g.ParameterError):
        g.ShardSystem(g.build_band_csr(1002, 8, 10, 1), grp, 0)
    with pytest.raises(g.UnsupportedError):
        g.ShardSystem(g.build_band_csr(1024, 8, 300, 1), grp, 1)
    grp.close()


def test_nccl_transport_world1_band():
    """A band CSR row block over the NCCL transport (one rank: the window is
    the whole matrix): the same bits as the unsharded solve."""
    A = g.build_band_csr(8192, 26, 300, 3)
    cfg = g.GadiConfig(alpha=3.0, xi=1e-20, u_r=g.Precision.Half, accum=g.Accum.Fp32,
                       inner=g.InnerSolverSpec(g.InnerMethod.Cg, 1e-12, 5, 30))
    full = g.CudaGadiSystem(A)
    xt = torch.empty(A.n_rows, dtype=torch.float64, device="cuda")
    b = torch.empty_like(xt)
    full.make_rhs(1, -1.0, 1.0, xt.data_ptr(), b.data_ptr())
    x1 = torch.empty_like(xt)
    rep1 = full.solve_device(b.data_ptr(), x1.data_ptr(), cfg)
    grp = g.ShardGroup.nccl(1, 0, g.nccl_unique_id())
    sh = g.ShardSystem(A, grp, 0)
    x2 = torch.empty_like(xt)
    rep2 = sh.solve_device(b.data_ptr(), x2.data_ptr(), cfg)
    torch.cuda.synchronize()
    assert rep2.outer_iters == rep1.outer_iters and rep2.status == rep1.status
    assert np.array_equal(bits(x2), bits(x1))
    sh.close()
    grp.close()
    full.close()
