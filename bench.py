#!/usr/bin/env python
"""GADI-IR time-to-1e-10 benchmark (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c3|c2|c4|c1|c5]

A step is one complete GADI-IR solve of the workload's system to relative
residual 1e-10 (xi = 1e-20): FP64 outer residual/update, inner CG on H and
GMRES on S on the device. Workloads (BASELINE.json configs):
  c3 (default, the north star's target): 3D convection-diffusion n=512
     (N = 134,217,728), beta=100, FP16 storage / FP32 arithmetic inner, FP64
     outer, alpha=0.22, omega=0.25, CG/GMRES(30) with eps=1e-12, max_inner=7
     (the fastest time-to-solution of an (alpha, omega, max_inner) sweep on B200).
  c2: n=256 (N = 16,777,216), beta=10, FP32 inner, alpha=0.11, omega=0.25, max_inner=10 (swept, round 2).
  c1: the reference's own CPU case: build_convdiff3d(32) (beta=1), FP16 inner
     through its default inner method (BandLU, lu_direct), alpha=0.1; the
     reference arm times its whole solve (measured, not projected).
x_true ~ U[-1,1) from the splitmix64 counter RNG (seed 1), b = A x_true in
binary64 on the device (the same generator the oracle uses).

value  = device time of one solve with b already in HBM (CUDA events inside
         the library, max over ranks), seconds; lower is better.
e2e    = the same solve through the C ABI gadi_cuda_solve with HOST buffers
         (pinned b in, x out; copies inside the timed region).
roofline = the inner CG sweep (SpMV + axpys + dots, SURVEY §8(d) B_CG =
         11 N s_r bytes per iteration) against MEASURED_PEAKS.json hbm_gbs.
Multi-GPU (torchrun, one rank per GPU; launched bare, --gpus N spawns the
ranks itself): the workload is partitioned over the ranks -- z-slabs of the
stencil grid, contiguous row blocks of the band CSR -- with
halo exchanges and rank-ordered reduction records over the library's CUDA IPC
transport (GADI_TRANSPORT=nccl: one NCCL communicator). Strong scaling: the
same problem at every N.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # BASELINE configs[0]: the reference's own build_convdiff3d(32) (beta = 1), x_true ~ U[0,1) seed 0,
    # FP16 inner through the reference's default inner method (BandLU, lu_direct), FP64 outer
    "c1": dict(n=32, beta=1.0, u_r=0, accum=0, method=0, alpha=0.1, eps=1e-2, max_inner=1000, restart=30,
               seed=0, lo=0.0, hi=1.0, s_r=4, name="convdiff3d n=32 beta=1 fp16 lu_direct inner (BandLU)"),
    "c3": dict(n=512, beta=100.0, u_r=0, accum=1, alpha=0.22, omega=0.25, eps=1e-12, max_inner=7, restart=30,
               seed=1, lo=-1.0, hi=1.0, s_r=2, name="convdiff3d n=512 beta=100 fp16-storage/fp32-accum inner"),
    "c2": dict(n=256, beta=10.0, u_r=1, accum=0, alpha=0.11, omega=0.25, eps=1e-12, max_inner=10, restart=30,
               seed=1, lo=-1.0, hi=1.0, s_r=4, name="convdiff3d n=256 beta=10 fp32 inner"),
    # BASELINE configs[3]: general nonsymmetric CSR, N = 2^24, 26 off-diagonals per row
    # uniform within +-4096 (seed 2), diagonal 1.1 x row abs sum; generated + split on the device
    "c4": dict(kind="band", N=1 << 24, k_off=26, band=4096, mseed=2, u_r=0, accum=1, alpha=4.0, eps=1e-12,
               max_inner=1, restart=30, seed=1, lo=-1.0, hi=1.0, s_r=2,
               name="band CSR N=2^24 27 nnz/row +-4096 fp16-storage/fp32-accum inner"),
}
# outer iterations the device solve needs for each workload (measured on B200,
# profiles/); used only to project the CPU reference's time-to-solution
OUTER_ITERS = {"c3": 442, "c2": 474, "c4": 28, "c1": 0}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("hbm_gbs", 6650.0), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = sorted(float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit())
        mx = max((float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()), default=None)
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for k, nm in enumerate(names):
                if len(r) > 4 + k and r[4 + k].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def c1_cpu_full(wl):
    """C1 fits the reference: time its whole solve (oracle/_ref, one core) on the
    same system, config and right-hand side -- measured, not projected."""
    from oracle import Config, Oracle, Reference
    o = Oracle()
    use_ref = Reference.available()
    R = Reference() if use_ref else o
    n = wl["n"]
    A = o.convdiff(n, 6.0, -1.0 - 1.0 / (2 * n + 2), -1.0 + 1.0 / (2 * n + 2))
    _, b = o.make_rhs(A, wl["seed"], wl["lo"], wl["hi"])
    cfg = Config.make(alpha=wl["alpha"], xi=1e-20, u_r=wl["u_r"], method=wl["method"])
    t = time.perf_counter()
    _, rep, _ = R.solve(A, b, cfg)
    dt = time.perf_counter() - t
    return {"value": dt, "unit": "s", "cores": 1, "kind": "reference" if use_ref else "port",
            "sample": (f"the whole C1 solve (build_convdiff3d(32), fp16 BandLU inner, alpha={wl['alpha']}): "
                       f"status {rep.status}, {rep.outer_iters} outer, measured (not projected)")}


def cpu_reference_sample(wl, full=False, outer=None):
    """Time the reference's own CPU implementation (oracle/_ref, compiled from
    the reference sources; else the oracle port) on a bounded sample of the
    workload and project it to the workload's size.

    The sample solves the same family at a size the host finishes in bounded
    time -- the stencil at n_s with the workload's r = beta h / 2, the band CSR
    at N_s rows with the same generator -- in the reference's FP32 Krylov mode
    (its FP16 Krylov overflows in the dots at these sizes) with the
    workload's alpha / eps / max_inner. hss_split runs once; gadi_ir_solve is
    then capped at k1 and at k2 outer steps and the two times are subtracted,
    so the one-time setup (CSR copy, split, regularize/prepare, the initial
    residuals) is counted once, not per step:

        per_outer_s = (t(k2) - t(k1)) / (k2 - k1)          at N_s
        setup_s     = t_split + t(k1) - k1 per_outer_s      at N_s
        value       = (N / N_s) (setup_s + outer_iters per_outer_s)

    outer_iters is the device solve's count on the workload (the same
    precision class converges within a few steps of it, tests/
    test_gpu_baseline_shapes.py). full=True (the reference arm) samples at the
    largest size that fits the host (n_s = 256, N_s = 2^21); the cpu_baseline
    leg of the default run uses n_s = 128 / N_s = 2^19 (about 30 s)."""
    if wl_key(wl) == "c1":
        return c1_cpu_full(wl)
    import psutil
    from oracle import CG, Config, Oracle, Reference
    o = Oracle()
    use_ref = Reference.available()
    big = full and psutil.virtual_memory().available > 48 * 2 ** 30
    if wl.get("kind") == "band":  # C4 cannot be split in host RAM
        ns, N_s, N_t = None, (1 << 21) if big else (1 << 19), wl["N"]
        A = o.band(N_s, wl["k_off"], wl["band"], wl["mseed"])
        r = 0.0
    else:
        ns = 256 if big else 128
        N_s, N_t = ns ** 3, wl["n"] ** 3
        r = wl["beta"] / (2.0 * (wl["n"] + 1.0))
        A = o.convdiff(ns, 6.0, -1.0 - r, -1.0 + r)
    _, b = o.make_rhs(A, wl["seed"], wl["lo"], wl["hi"])
    k1, k2 = (1, 2) if big else (1, 3)
    cfg = Config.make(alpha=wl["alpha"], omega=wl.get("omega", 1.0), xi=1e-20, u_r=1, method=CG, tol_epsilon=wl["eps"],
                      max_inner_iters=wl["max_inner"], restart=wl["restart"])
    if use_ref:
        t_split, t1, t2, o1, o2 = Reference().solve_steps_timed(A, b, cfg, k1, k2)
    else:  # the port has no separate split: both capped solves carry it
        ts = []
        for k in (k1, k2):
            cfg.max_outer_iters = k
            t = time.perf_counter()
            _, rep, _ = o.solve(A, b, cfg)
            ts.append(time.perf_counter() - t)
        t_split, t1, t2, o1, o2 = 0.0, ts[0], ts[1], k1, k2
    per_outer = (t2 - t1) / max(1, o2 - o1)
    setup = t_split + t1 - o1 * per_outer
    scale = N_t / N_s
    outer = outer or OUTER_ITERS[wl_key(wl)]
    proj = scale * (setup + outer * per_outer)
    what = (f"band CSR N={N_s}" if ns is None else f"n={ns} (N={N_s}) with r={r:.5f}")
    return {
        "value": proj, "unit": "s", "cores": 1, "kind": "reference" if use_ref else "port",
        "setup_s": setup, "per_outer_s": per_outer, "sample_rows": N_s, "scale": scale, "outer_iters": outer,
        "ns_per_row_per_outer": per_outer / N_s * 1e9,
        "formula": "value = scale * (setup_s + outer_iters * per_outer_s); per_outer_s = (t(k2)-t(k1))/(k2-k1)",
        "sample": (f"reference gadi_ir_solve (fp32 CG/GMRES, max_inner={wl['max_inner']}) on {what}: hss_split "
                   f"{t_split:.2f} s, solve capped at {o1} outer {t1:.2f} s, at {o2} outer {t2:.2f} s -> "
                   f"{per_outer:.3f} s per outer step, {setup:.2f} s setup; projected x{scale:g} rows and "
                   f"{outer} outer steps (single-threaded: the reference has no intra-solve parallelism)"),
    }


def c5_data():
    """BASELINE configs[4]: m = 4096 pairs, log10 N ~ U[4,8], alpha = 0.5 N^(-1/3)
    (1 + 0.05 N(0,1)) (seed 3); 65,536 query sizes log10 N ~ U[4,8]. Sizes are
    rounded to integers (the reference's index_t sizes) and made unique."""
    import numpy as np
    rng = np.random.default_rng(3)
    sizes = np.unique(np.round(10.0 ** rng.uniform(4, 8, 4096 + 64)))[:4096]
    alphas = 0.5 * sizes ** (-1.0 / 3.0) * (1.0 + 0.05 * rng.standard_normal(len(sizes)))
    q = np.round(10.0 ** rng.uniform(4, 8, 65536))
    var = max(float(np.mean((alphas - alphas.mean()) ** 2)), 1e-8)
    return sizes, alphas, q, (var, 1.0, 1e-4)  # sigma_f2 = var(y) (the grid's middle), l = 1, sn2 = 1e-4


def run_c5(args, rank, world):
    """GPR alpha predictor (BASELINE configs[4]): one step = fit (fixed hypers,
    m x m Gram + Cholesky) + predict 65,536 queries (mean + std)."""
    import numpy as np
    sizes, alphas, q, fixed = c5_data()
    metric = "GPR fit+predict time (m=4096, q=65536)"
    cfg = {"workload": "GPR alpha predictor m=4096 q=65536", "m": len(sizes), "q": len(q),
           "sigma_f2": fixed[0], "length": fixed[1], "sigma_n2": fixed[2]}
    if args.impl == "reference":
        if rank == 0:
            cb = c5_cpu_sample(sizes, alphas, q, fixed)
            print(json.dumps({"impl": "reference", "metric": metric, "value": cb["value"], "unit": "s",
                              "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                              "higher_is_better": False, "dtype": "f64", "data": "synthetic", "config": cfg,
                              "cpu_baseline": cb, "e2e": {"value": cb["value"], "unit": "s",
                                                          "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return
    import torch
    import paper_2501_04229_b200 as g
    one_gpu = os.environ.get("GADI_BENCH_ONE_GPU") == "1"  # dry run: all ranks on device 0
    dev = 0 if one_gpu else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(dev)
    tm = {}
    if world > 1:
        # N > 1: every rank fits (12 ms, replicated) and predicts its contiguous slice of the
        # queries; the slices are gathered in rank order (control plane: gloo)
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        cfg["parallelism"] = f"queries/{world} (fit replicated)"

    def step():
        m = g.gpr_fit(sizes, alphas, fixed=fixed, device=dev)
        out = m.predict(q) if world == 1 else m.predict_sharded(q, rank, world)
        tm.update(m.timings())
        m.close()
        return out

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    l0 = 0
    t = time.perf_counter()
    var_ms = []
    for _ in range(args.steps):
        mean, sd = step()
        var_ms.append(tm["variance_ms"])
        l0 += tm["launches"]
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / args.steps
    if world > 1:  # the step ends with a gather, so every rank's clock covers the slowest rank; take the max
        tt = torch.tensor([dt], dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
    mq, nq = len(sizes), len(q)
    mp = (mq + 255) // 256 * 256
    # the variance GEMM D = X K_*: lower-triangular X (mp x mp) times mp x q, three fp16 MMAs per product
    tens_flops = 3.0 * 2.0 * (mp * (mp + 256) / 2.0) * ((nq + 255) // 256 * 256)
    vms = sum(var_ms) / len(var_ms)
    peak = 1590.0
    pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peak_kind = "fallback"
    if os.path.exists(pk):
        with open(pk) as f:
            peak = json.load(f).get("bf16_tflops", peak)
        peak_kind = "measured (bf16 burst)"
    ach = tens_flops / (vms / 1e3) / 1e12 if tm["variance_path"] == "tensor" else None
    out = {"metric": metric, "value": dt, "unit": "s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": False,
           "scaling": "strong" if world > 1 else "weak",
           "vs_baseline": None, "dtype": "f64 fit / f16 hi+lo tensor-core variances (f32 accumulate)",
           "data": "synthetic", "config": cfg,
           "e2e": {"value": dt, "unit": "s", "h2d_bytes_per_step": 8 * (2 * mq + nq),
                   "d2h_bytes_per_step": 16 * nq},
           "gpu_launches": int(l0),
           "roofline": {"bound": "tensor", "kernel": "k_var_umma (variances: X K_* on tcgen05, fp16 hi/lo, 3 MMAs per product)",
                        "achieved": ach, "peak": peak, "peak_kind": peak_kind, "unit": "TFLOP/s",
                        "frac": ach / peak if ach else None, "traffic": None,
                        "tensor_flops_per_launch": tens_flops, "useful_flops": float(mp) * mp * nq,
                        "kernel_ms": vms},
           "phases_ms": {"fit": tm["fit_ms"], "inverse_factor": tm["inverse_ms"], "variance": vms,
                         "variance_path": tm["variance_path"]},
           "note": "host-timed end to end (inputs/outputs are host arrays); hand-written kernels only "
                   "(libgadi_cuda.so links libcudart alone)",
           "flops": {"cholesky": mq ** 3 / 3, "trsm": mq ** 2 * nq},
           "prediction_sample": {"mean_min": float(mean.min()), "mean_max": float(mean.max()),
                                 "sd_max": float(sd.max())}}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = c5_cpu_sample(sizes, alphas, q, fixed)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def c5_cpu_sample(sizes, alphas, q, fixed):
    """The oracle restatement of fit/predict (gpr.cpp:72-169; the reference's
    gpr.cpp needs Eigen, absent here) on one host core: the full fit plus 256
    of the 65,536 queries, projected linearly in the query count."""
    from oracle import Oracle
    o = Oracle()
    t = time.perf_counter()
    o.gpr(sizes, alphas, q[:1], fixed=fixed)
    t_fit = time.perf_counter() - t
    t = time.perf_counter()
    o.gpr(sizes, alphas, q[:257], fixed=fixed)
    t_q = (time.perf_counter() - t - t_fit) / 256
    proj = t_fit + t_q * len(q)
    return {"value": proj, "unit": "s", "cores": 1, "kind": "port",
            "sample": f"fit m={len(sizes)} ({t_fit:.1f} s) + 256 queries ({t_q * 1e3:.1f} ms each), "
                      f"projected to {len(q)} queries"}


def wl_key(wl):
    for k, v in WORKLOADS.items():
        if v is wl:
            return k
    return "c3"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3", choices=list(WORKLOADS) + ["c5"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # launched bare: start one rank per GPU ourselves (the launch the driver uses)
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.workload == "c5":
        return run_c5(args, rank, world)
    wl = WORKLOADS[args.workload]
    metric = "GADI-IR time-to-1e-10 residual"
    band = wl.get("kind") == "band"
    Nw = wl["N"] if band else wl["n"] ** 3
    lu = wl.get("method") == 0
    cfg_json = {"workload": wl["name"], "N": Nw, "alpha": wl["alpha"], "omega": wl.get("omega", 1.0),
                "inner": "lu_direct(H, S)" if lu else "cg(H)/gmres(S)",
                "max_inner": wl["max_inner"], "tol_epsilon": wl["eps"], "xi": 1e-20,
                "l2": "inputs larger than L2 (x, b: 8N bytes each)",
                "parallelism": "single"}
    # the stencil shards into z-slabs, the band CSR into row blocks (NCCL,
    # strong scaling: the same problem at every N)
    sharded = world > 1
    if world > 1:
        cfg_json["parallelism"] = f"rowblock{world}" if band else f"zslab{world}"
    if band:
        cfg_json.update(k_off=wl["k_off"], band=wl["band"], matrix_seed=wl["mseed"])
    else:
        cfg_json.update(n=wl["n"], beta=wl["beta"])

    if args.impl == "reference":
        if rank != 0:
            return
        cb = cpu_reference_sample(wl, full=True)
        print(json.dumps({"impl": "reference", "metric": metric, "value": cb["value"], "unit": "s",
                          "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                          "higher_is_better": False, "dtype": "f64", "data": "synthetic",
                          "config": cfg_json, "cpu_baseline": cb,
                          "e2e": {"value": cb["value"], "unit": "s", "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}), flush=True)
        return

    import torch
    import paper_2501_04229_b200 as g

    if os.environ.get("GADI_BENCH_ONE_GPU"):  # dry run of the multi-rank path on one GPU (IPC transport only)
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        # control plane only (barriers, a few scalars, the transport's rendezvous): gloo on the host.
        # The data plane is the library's own transport below.
        dist.init_process_group("gloo")
    if band:
        S = g.build_band_csr(wl["N"], wl["k_off"], wl["band"], wl["mseed"])
    else:
        S = g.build_convdiff3d(wl["n"], beta=wl["beta"])
    grp = None
    if sharded:
        # one rank per process: CUDA IPC on a node (peer-mapped staging buffers, interprocess events,
        # one-shot record gathers over NVLink), or NCCL with GADI_TRANSPORT=nccl
        transport = os.environ.get("GADI_TRANSPORT", "ipc")
        if transport == "nccl":
            obj = [g.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            grp = g.ShardGroup.nccl(world, rank, obj[0])
        else:
            grp = g.ShardGroup.ipc(world, rank, f"/gadi_bench_{os.environ.get('MASTER_PORT', '0')}_{os.getppid()}")
        cfg_json["transport"] = transport
        sysx = g.ShardSystem(S, grp, rank, device=local)
    else:
        sysx = g.CudaGadiSystem(S, device=local)
    N = sysx.n  # this rank's rows
    xt = torch.empty(N, dtype=torch.float64, device="cuda")
    b = torch.empty_like(xt)
    seed = wl["seed"] if (sharded or world == 1) else wl["seed"] + rank
    sysx.make_rhs(seed, wl["lo"], wl["hi"], xt.data_ptr(), b.data_ptr())  # collective on shards
    torch.cuda.synchronize()
    b_h = b.cpu().pin_memory()
    x_h = torch.empty(N, dtype=torch.float64).pin_memory()
    cfg = g.GadiConfig(alpha=wl["alpha"], omega=wl.get("omega", 1.0), xi=1e-20, u_r=g.Precision(wl["u_r"]),
                       accum=g.Accum(wl["accum"]),
                       inner=g.InnerSolverSpec(g.InnerMethod(wl.get("method", 1)), wl["eps"], wl["max_inner"],
                                               wl["restart"]))
    b_np = b_h.numpy()
    x_np = x_h.numpy()

    def step():
        # every timed solve re-runs prepare (operators, and the factorizations for lu_direct),
        # as the reference's gadi_ir_solve does on each call (solver.cpp:75, 199-208)
        sysx.reset()
        return sysx.solve_into(b_np, x_np, cfg)

    for _ in range(args.warmup):
        step()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    reps = []
    l0 = g.lib().gadi_cuda_launch_count(sysx._h)
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        for _ in range(args.steps):
            reps.append(step())
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    launches = g.lib().gadi_cuda_launch_count(sysx._h) - l0
    if dist:
        dist.barrier()
    solve_s = sum(r.solve_ms for r in reps) / len(reps) / 1e3
    e2e_s = sum(r.e2e_ms for r in reps) / len(reps) / 1e3
    h_ms = sum(r.h_ms for r in reps)
    h_it = sum(r.h_iters for r in reps)
    ok = all(r.status == g.SolveStatus.Converged for r in reps)
    x = torch.from_numpy(x_np).cuda()
    ss = torch.stack([torch.sum((x - xt) ** 2), torch.sum(xt ** 2)]).cpu()
    if sharded:
        dist.all_reduce(ss)
    ferr = (ss[0].sqrt() / ss[1].sqrt()).item()
    if dist:
        t = torch.tensor([solve_s, e2e_s], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        solve_s, e2e_s = t.tolist()
    peak, peak_kind = load_peaks()
    # inner CG sweep: B_CG = 11 N s_r bytes per iteration; a
    # sparse H adds, per SpMV, nnz(H) (s_r value + index) + the row lengths. The
    # index is what the SELL image stores: a 2-byte column offset when the band
    # is below 2^15 (configs[3]: +-4096), else a 4-byte column; row lengths are
    # 2 bytes per row (SURVEY's 6 B/nnz int32-CSR figure would overstate it)
    bytes_it = 11 * N * wl["s_r"]
    if band:
        idx_bytes = 2 if wl["band"] < 32768 else 4
        bytes_it += sysx.nnz()[1] * (wl["s_r"] + idx_bytes) + 2 * N
    cg_gbs = bytes_it * h_it / (h_ms / 1e3) / 1e9 if h_ms > 0 else None
    roof_kernel = ("inner CG iteration (p-update, SELL spmv + p.q, axpys + dots)" if band
                   else "inner CG iteration (spmv+p-update, axpys+dots)")
    if lu:  # one BandLU solve reads the factor band once: N (kl + (kl+ku) + 1) binary32 values (n^2 bands)
        kl = wl["n"] ** 2
        bytes_it = N * (kl + 2 * kl + 1) * 4
        n_solves = sum(r.outer_iters for r in reps)
        cg_gbs = bytes_it * n_solves / (h_ms / 1e3) / 1e9 if h_ms > 0 else None
        roof_kernel = "BandLU solve of H (forward + back sweeps over the factor band, k_lu_pipe)"
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"traffic_{args.workload}.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get("cg_iteration_dram_bytes")
    out = {
        "metric": metric, "value": solve_s, "unit": "s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": solve_s * 1e3, "higher_is_better": False,
        "scaling": "strong" if sharded else "weak",
        "vs_baseline": None, "dtype": "f64 outer / " + ("f16 (every op rounded to binary16)" if lu else
                                                       "f16 storage, f32 arithmetic" if wl["u_r"] == 0 else "f32")
        + " inner", "data": "synthetic (seeded splitmix64 x_true, b = A x_true)", "config": cfg_json,
        "e2e": {"value": e2e_s, "unit": "s", "h2d_bytes_per_step": int(reps[0].h2d_bytes),
                "d2h_bytes_per_step": int(reps[0].d2h_bytes)},
        "roofline": {"bound": "hbm", "kernel": roof_kernel,
                     "achieved": cg_gbs, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": (cg_gbs / peak) if cg_gbs else None, "traffic": traffic if world == 1 else None,
                     "algorithmic_bytes_per_iter": bytes_it, "per": "GPU (rank 0's shard)" if sharded else "GPU"},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "solve": {"converged": ok, "outer_iters": reps[0].outer_iters, "final_rres": reps[0].final_rres,
                  "forward_rel_err": ferr, "cg_iters": reps[0].h_iters, "gmres_iters": reps[0].s_iters,
                  "h_ms": reps[0].h_ms, "s_ms": reps[0].s_ms, "outer_ms": reps[0].outer_ms,
                  "wall_s_per_step": wall / args.steps},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_reference_sample(wl, outer=reps[0].outer_iters)
    if rank == 0:
        print(json.dumps(out), flush=True)
    sysx.close()
    if grp is not None:
        grp.close()
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
