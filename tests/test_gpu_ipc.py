"""The CUDA IPC transport (gadi_group_ipc, csrc/gadi_dist.cuh IpcComm): one
rank per PROCESS, 2 and 4 processes sharing this one GPU -- what NCCL refuses
("duplicate GPU") and what bench.py --gpus N launches on a node. Each rank
solves its z-slab / row block collectively; the gathered solution, the
iteration counts and the residual history must equal the one-device solve bit
for bit (every dot is the single-device pairwise tree, folded in rank order).

No kernel of the transport waits on another rank (stream waits on
interprocess events + a host barrier in shared memory), so processes that
time-slice one GPU make progress."""
import multiprocessing as mp
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _rank_main(rank, world, name, kind, q):
    try:
        sys.path.insert(0, ROOT)
        import torch
        import paper_2501_04229_b200 as g
        torch.cuda.set_device(0)
        if kind == "stencil":
            A = g.build_convdiff3d(32, r=100.0 / (2.0 * 513.0))
            cfg = g.GadiConfig(alpha=0.5, xi=1e-20, u_r=g.Precision.Half, accum=g.Accum.Fp32, stall_window=400,
                               inner=g.InnerSolverSpec(g.InnerMethod.Cg, 1e-12, 5, 30))
        elif kind == "stencil_f32":
            A = g.build_convdiff3d(16)
            cfg = g.GadiConfig(alpha=0.1, xi=1e-20, u_r=g.Precision.Single,
                               inner=g.InnerSolverSpec(g.InnerMethod.Cg, 1e-12, 50, 30))
        else:
            A = g.build_band_csr(8192, 26, 300, 3)
            cfg = g.GadiConfig(alpha=3.0, xi=1e-20, u_r=g.Precision.Half, accum=g.Accum.Fp32,
                               inner=g.InnerSolverSpec(g.InnerMethod.Cg, 1e-12, 5, 30))
        grp = g.ShardGroup.ipc(world, rank, name)
        sh = g.ShardSystem(A, grp, rank)
        xt = torch.empty(sh.n, dtype=torch.float64, device="cuda")
        b = torch.empty_like(xt)
        x = torch.empty_like(xt)
        sh.make_rhs(1, -1.0, 1.0, xt.data_ptr(), b.data_ptr())
        rep = sh.solve_device(b.data_ptr(), x.data_ptr(), cfg)
        rep2 = sh.solve_device(b.data_ptr(), x.data_ptr(), cfg)  # a second solve on the same communicator
        torch.cuda.synchronize()
        q.put((rank, sh.first_row, x.cpu().numpy(), int(rep.status), rep.outer_iters, rep.inner_iter_totals,
               np.array(rep.rel_residual_history), rep2.outer_iters))
        sh.close()
        grp.close()
    except Exception as e:  # surface the failure in the parent
        import traceback
        q.put((rank, -1, traceback.format_exc(), repr(e)))


@pytest.mark.parametrize("kind,world", [("stencil", 2), ("stencil", 4), ("band", 2), ("stencil_f32", 2)])
def test_ipc_ranks_equal_one_device(kind, world):
    import torch
    import paper_2501_04229_b200 as g
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    name = f"/gadi_ipc_test_{os.getpid()}_{kind}_{world}"
    procs = [ctx.Process(target=_rank_main, args=(r, world, name, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = []
    for _ in range(world):
        outs.append(q.get(timeout=600))
    for p in procs:
        p.join(timeout=120)
    for o in outs:
        assert o[1] != -1, o[2]
    outs.sort(key=lambda o: o[0])
    x = np.concatenate([o[2] for o in outs])
    # the same problem on one device in this process
    if kind == "stencil":
        A = g.build_convdiff3d(32, r=100.0 / (2.0 * 513.0))
        cfg = g.GadiConfig(alpha=0.5, xi=1e-20, u_r=g.Precision.Half, accum=g.Accum.Fp32, stall_window=400,
                           inner=g.InnerSolverSpec(g.InnerMethod.Cg, 1e-12, 5, 30))
    elif kind == "stencil_f32":
        A = g.build_convdiff3d(16)
        cfg = g.GadiConfig(alpha=0.1, xi=1e-20, u_r=g.Precision.Single,
                           inner=g.InnerSolverSpec(g.InnerMethod.Cg, 1e-12, 50, 30))
    else:
        A = g.build_band_csr(8192, 26, 300, 3)
        cfg = g.GadiConfig(alpha=3.0, xi=1e-20, u_r=g.Precision.Half, accum=g.Accum.Fp32,
                           inner=g.InnerSolverSpec(g.InnerMethod.Cg, 1e-12, 5, 30))
    full = g.CudaGadiSystem(A)
    xt = torch.empty(A.n_rows, dtype=torch.float64, device="cuda")
    b = torch.empty_like(xt)
    x1 = torch.empty_like(xt)
    full.make_rhs(1, -1.0, 1.0, xt.data_ptr(), b.data_ptr())
    rep1 = full.solve_device(b.data_ptr(), x1.data_ptr(), cfg)
    torch.cuda.synchronize()
    full.close()
    assert int(rep1.status) == 0
    for o in outs:
        assert (o[3], o[4], o[5]) == (int(rep1.status), rep1.outer_iters, rep1.inner_iter_totals)
        assert np.array_equal(o[6].view(np.int64), np.array(rep1.rel_residual_history).view(np.int64))
        assert o[7] == rep1.outer_iters
    assert np.array_equal(x.view(np.int64), x1.cpu().numpy().view(np.int64))
