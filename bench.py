"""Benchmark of the B200 solve phase: preconditioned CGLS iterations/s.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config 1]

A step is one preconditioned CGLS iteration of pcgls (sv.py:202-241) -- one
product with A and A^T, one row-splitting preconditioner application, the
dots and the scalar recursion -- on the BASELINE.json workload (config 1:
256^2 grid, n = 65,536, m = 98,304, cg(2) coupling solve because s = 32,768
exceeds the dense cap, mu = 1.0).  Inputs are the seeded
synthetic generators of paper_2603_28642_b200/workloads.py.

The timed region is device time (CUDA events on the solver's stream) of K
iterations run as replays of the captured iteration graph, with the L2
flushed before every iteration outside the bracket; `e2e` is the same metric
through the public API (pcgls with host buffers: H2D of b, D2H of x inside).
Under torchrun each rank solves its own right-hand side on its own GPU
(replicas, weak scaling; no collective on the data path); times are the max
over ranks.  --impl reference times the CPU oracle port of the reference's
pcgls on the same workload (the reference itself is pure Python/numpy and
cannot travel to the GPU box).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

FALLBACK_HBM_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--mu", type=float, default=1.0)
    ap.add_argument("--mode", default=None, help="coupling solve: dense | cg | identity")
    ap.add_argument("--grid", type=int, default=256, help="config 1 grid side")
    ap.add_argument("--n", type=int, default=None, help="override n for configs 0/2/3/4")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--no-tol", action="store_true", help="skip the time-to-tolerance run")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--batch", type=int, default=8,
                    help="also time this many concurrent RHS per GPU through pcgls_batch (0: skip)")
    ap.add_argument("--blas-threads", type=int, default=1,
                    help="reproduce the reference's OpenBLAS dot order at this many threads "
                         "(OPENBLAS_NUM_THREADS; 1 = the pinned single-thread order)")
    ap.add_argument("--partition", default="replicas", choices=["replicas", "rows"],
                    help="N>1: replicas (one RHS per GPU, weak) or rows (one RHS, A row-partitioned, "
                         "NCCL allreduce of A^T r, strong)")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


# ---------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------


def make_workload(args, rank):
    from paper_2603_28642_b200 import workloads as W

    cfgid = args.config
    st = dict(W.SETTINGS[cfgid])
    t0 = time.perf_counter()
    if cfgid == 1:
        A, b = W.config1(seed=1, g=args.grid)
        name = f"config1: {args.grid}x{args.grid} grid LS, n={A.ncols}, m={A.nrows}"
    elif cfgid == 0:
        A, b = W.config0(seed=0, **({} if args.n is None else dict(n=args.n, m=3 * args.n // 2)))
        name = f"config0: random sparse LS, n={A.ncols}, m={A.nrows}"
    elif cfgid == 2:
        A, b = W.config2(seed=2, **({} if args.n is None else dict(n=args.n)))
        name = f"config2: sparse + 100 dense rows, n={A.ncols}, m={A.nrows}"
    elif cfgid == 3:
        A, b = W.config3(seed=3, n=args.n or 100_000)
        name = f"config3: ill-conditioned random LS, n={A.ncols}, m={A.nrows}"
    else:
        A, B = W.config4(seed=4, n=args.n or 1_000_000, nrhs=max(1, rank + 1))
        b = B[rank]
        name = f"config4 structure: n={A.ncols}, m={A.nrows}"
    if rank > 0 and cfgid != 4:
        # replicas: every rank solves its own right-hand side
        b = b + 1e-3 * np.random.default_rng(1000 + rank).standard_normal(len(b))
    t_gen = time.perf_counter() - t0
    return A, b, st, name, t_gen


def setup(args, A, st):
    import paper_2603_28642_b200 as P

    times = {}
    t0 = time.perf_counter()
    if st["scale"]:
        S, _ = P.column_scale(A)
    else:
        S = A
    times["column_scale_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    f = P.ilup_factorize(S, P.IlupParams(p=st["p"], tau=st["tau"], mu=args.mu))
    times["ilup_host_s"] = time.perf_counter() - t0
    mode = args.mode or st["s_mode"]
    if mode == "dense" and f.L2.nrows > 20000:
        mode = "cg"  # the reference CLI's fallback (cli.py:68-78)
    t0 = time.perf_counter()
    pre = P.build_preconditioner(f, s_mode=P.SMode(mode))
    times["build_preconditioner_s"] = time.perf_counter() - t0
    return S, f, pre, mode, times


# ---------------------------------------------------------------------------
# clocks
# ---------------------------------------------------------------------------


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.thread.join(timeout=2)

    def summary(self):
        rows = [r for r in self.rows if len(r) >= 8]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower() == "active"})
        loaded = [v for v in sm if mx and v > 0.5 * max(mx)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------
# roofline bookkeeping (int32 indices, f64 values)
# ---------------------------------------------------------------------------


def tri_bytes(nnz, n):
    return 12 * nnz + 4 * (n + 1) + 16 * n


def trsv_bytes_per_iteration(pre, mode):
    f = pre.factors
    n, s = f.U.ncols, f.L2.nrows
    l1 = tri_bytes(f.L1.nnz, n)
    u = tri_bytes(f.U.nnz, n)
    k = pre.cg_iters
    if s == 0:
        return l1 + u, {"L1": 1, "L1T": 0, "U": 1}
    if mode == "cg":
        counts = {"L1": 2 + k, "L1T": 1 + k, "U": 1}
    elif mode == "identity":
        counts = {"L1": 2, "L1T": 1, "U": 1}
    else:  # dense: explicit Y, one L1 solve
        counts = {"L1": 1, "L1T": 0, "U": 1}
    return (counts["L1"] + counts["L1T"]) * l1 + counts["U"] * u, counts


def measured_peak():
    path = os.path.join(HERE, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return FALLBACK_HBM_GBS, "fallback"


def ncu_traffic():
    """DRAM bytes (read + write) per iteration of the dominant kernel class,
    summed over the iteration's solves, from the committed ncu capture
    (profiles/ncu_trsv_r01.json), or None."""
    path = os.path.join(HERE, "profiles", "ncu_trsv_r01.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return d.get("dram_bytes_per_iteration"), d.get("source")
    except (OSError, ValueError):
        return None, None


# ---------------------------------------------------------------------------
# arms
# ---------------------------------------------------------------------------


CPU_THREADS_NOTE = ("one core: the reference solve is sequential (triangular solves, np.add.at / reduceat scatters in numpy); only its BLAS dots could use more threads, and the port runs them in the reference's one-thread OpenBLAS order (--blas-threads T selects the T-thread order)")


def cpu_oracle_rate(S, pre, b, norm_a, budget_s, max_iters_cap=400):
    """Oracle port of pcgls (oracle/oracle.py), single thread, fixed-iteration
    run sized to roughly budget_s seconds; returns (iters/s, iters, seconds)."""
    from oracle import oracle as O

    op = O.OraclePreconditioner.from_reference(pre)
    O.set_blas_threads(int(os.environ.get("RSB_BLAS_THREADS", "1")))
    t0 = time.perf_counter()
    O.pcgls(S, b, op, norm_a, delta=1e-300, max_iters=2)
    probe = max(time.perf_counter() - t0, 1e-4) / 2
    k = int(max(3, min(max_iters_cap, budget_s / probe)))
    t0 = time.perf_counter()
    O.pcgls(S, b, op, norm_a, delta=1e-300, max_iters=k)
    dt = time.perf_counter() - t0
    return k / dt, k, dt


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    from oracle import oracle as O

    O.set_blas_threads(args.blas_threads)

    A, b, st, name, _ = make_workload(args, 0)
    S, f, pre, mode, _ = setup(args, A, st)
    norm_a = O.power_method_norm2(S, 100, args.config)
    # warmup + K steps, each step one iteration; bounded sample
    op = O.OraclePreconditioner.from_reference(pre)
    O.pcgls(S, b, op, norm_a, delta=1e-300, max_iters=max(1, min(args.warmup, 3)))
    k = args.steps
    t0 = time.perf_counter()
    O.pcgls(S, b, op, norm_a, delta=1e-300, max_iters=k)
    dt = time.perf_counter() - t0
    value = k / dt
    line = {
        "impl": "reference", "metric": "preconditioned CGLS iterations/s", "value": value,
        "unit": "iter/s", "n_gpus": args.gpus, "steps": k, "warmup": args.warmup,
        "ms_per_step": 1e3 * dt / k, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded generators, workloads.py)",
        "config": {"workload": name, "mu": args.mu, "coupling": mode, "p": st["p"], "tau": st["tau"]},
        "cpu_baseline": {"value": value, "unit": "iter/s", "cores": 1, "kind": "port",
                         "sample": f"{k} fixed iterations (delta=1e-300) of the oracle port of pcgls",
                         "threads": CPU_THREADS_NOTE},
        "e2e": {"value": value, "unit": "iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_b200(args):
    rank, world, local = dist_env()
    os.environ.setdefault("RSB_DEVICE", str(local))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as tdist

        torch.cuda.set_device(local)
        tdist.init_process_group("nccl")
        dist = (torch, tdist)

    def barrier_max(x):
        if dist is None:
            return x
        torch, tdist = dist
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        return float(t.item())

    def barrier():
        if dist is not None:
            dist[1].barrier()

    import paper_2603_28642_b200 as P
    from paper_2603_28642_b200 import _lib as L
    from paper_2603_28642_b200.device import (DeviceBuffer, PinnedBuffer, device_matrix,
                                              device_preconditioner, device_solver, get_context)

    A, b, st, name, t_gen = make_workload(args, rank)
    S, f, pre, mode, times = setup(args, A, st)
    ctx = get_context()
    t0 = time.perf_counter()
    dA = device_matrix(S, ctx)
    dpre = device_preconditioner(pre, ctx)
    solver = device_solver(dA, dpre)
    lv_l1 = dpre.L1.levels(L.TRI_LOWER_UNIT)
    lv_u = dpre.U.levels(L.TRI_UPPER)
    variants = {"L1": dpre.L1.variant(L.TRI_LOWER_UNIT), "L1T": dpre.L1.variant(L.TRI_LOWER_T_UNIT),
                "U": dpre.U.variant(L.TRI_UPPER)}
    times["upload_and_analysis_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    norm_a = P.power_method_norm2(S, 100, args.config)
    times["power_method_device_s"] = time.perf_counter() - t0

    K, Wm = args.steps, args.warmup
    # ---- device-resident timed region
    bdev = DeviceBuffer(ctx, len(b))
    bdev.upload(b)
    cfg = solver.cfg_struct(norm_a, 1e-300, Wm + K + 8, 5, False)
    status = solver.start(bdev.ptr, L.RSB_DEVICE, cfg)
    if status != 0:
        raise RuntimeError(f"solver stopped at start (status {status})")
    solver.iterate(Wm)
    it_ms, tri_ms = np.zeros(1), np.zeros(1)
    tri_launches, kpi, st_out = (np.zeros(1, dtype=np.int64) for _ in range(3))
    barrier()
    with ClockSampler(local) as clocks:
        st_c = np.zeros(1, dtype=np.int32)
        L.check(L.lib().rsb_solver_bench(solver.h, K, 0 if args.no_flush else 1,
                                         it_ms.ctypes.data_as(L.f64p), tri_ms.ctypes.data_as(L.f64p),
                                         tri_launches.ctypes.data_as(L.i64p), kpi.ctypes.data_as(L.i64p),
                                         st_c.ctypes.data_as(L.ctypes.POINTER(L.ctypes.c_int))))
    barrier()
    if st_c[0] != 0:
        raise RuntimeError(f"solver left the fixed-iteration run early (status {st_c[0]})")
    iter_ms_max = barrier_max(float(it_ms[0]))
    value = world * K / (iter_ms_max / 1e3)

    # ---- end to end through the public API (host buffers, copies inside)
    bpin = PinnedBuffer(len(b))
    bpin.array[:] = b
    e2e_cfg = P.CglsConfig(norm_A=norm_a, delta=1e-300, max_iters=K)
    P.pcgls(S, bpin.array, pre, P.CglsConfig(norm_A=norm_a, delta=1e-300, max_iters=max(1, Wm)))
    barrier()
    t0 = time.perf_counter()
    x, rep = P.pcgls(S, bpin.array, pre, e2e_cfg)
    e2e_s = barrier_max(time.perf_counter() - t0)
    e2e = world * rep.its / e2e_s if not rep.converged else world * K / e2e_s

    # ---- several independent RHS per GPU, solved concurrently
    batch = None
    if args.batch > 1:
        rng = np.random.default_rng(77 + rank)
        Bm = np.stack([b] + [b + 1e-3 * rng.standard_normal(len(b)) for _ in range(args.batch - 1)])
        P.pcgls_batch(S, Bm, pre, P.CglsConfig(norm_A=norm_a, delta=1e-300, max_iters=max(1, Wm)))
        barrier()
        t0 = time.perf_counter()
        _, breps = P.pcgls_batch(S, Bm, pre, e2e_cfg)
        b_s = barrier_max(time.perf_counter() - t0)
        its = sum(K if r.converged else r.its for r in breps)
        batch = {"rhs_per_gpu": args.batch, "value": world * its / b_s, "unit": "RHS-iter/s",
                 "seconds": b_s,
                 "call": f"pcgls_batch(A, B[{args.batch} x m] host, pre, CglsConfig(delta=1e-300, "
                         f"max_iters={K})): one stream + workspace per RHS, shared A and factors; all RHS "
                         f"iterate concurrently when the solves are single-CTA, two at a time when "
                         f"they are grid-wide (each fills most of the GPU)"}

    # ---- time to tolerance (config delta), device path, reported alongside
    tol = None
    if not args.no_tol:
        t0 = time.perf_counter()
        nrm = P.power_method_norm2(S, 100, args.config)
        _, rtol = P.pcgls(S, b, pre, P.CglsConfig(norm_A=nrm, delta=st["delta"], max_iters=st["max_iters"]))
        tol = {"seconds": barrier_max(time.perf_counter() - t0), "its": rtol.its,
               "converged": rtol.converged, "breakdown": rtol.breakdown, "delta": st["delta"],
               "ratio_pt_final": rtol.ratio_pt_final,
               "grad_ratio": rtol.gradient_norm_final / (nrm * rtol.residual_norm_final)
               if rtol.residual_norm_final > 0 else 0.0,
               "includes": "power method (100 its) + pcgls to delta, host b in / x out"}

    if rank != 0:
        return
    # ---- roofline of the dominant kernel class (the triangular solves)
    tbytes, counts = trsv_bytes_per_iteration(pre, mode)
    ntri = int(tri_launches[0])
    achieved = (tbytes * K) / (tri_ms[0] / 1e3) / 1e9
    peak, peak_kind = measured_peak()
    traffic, traffic_src = ncu_traffic()
    if not (args.config == 1 and args.grid == 256 and args.mu == 1.0 and mode == "cg"):
        traffic, traffic_src = None, "no ncu capture committed for this workload"
    cpu = None
    if world == 1:
        rate, kc, dtc = cpu_oracle_rate(S, pre, b, norm_a, args.cpu_seconds)
        cpu = {"value": rate, "unit": "iter/s", "cores": 1, "kind": "port",
               "sample": f"{kc} fixed iterations (delta=1e-300) of the oracle port of pcgls on the same "
                         f"workload, {dtc:.1f} s, host has {os.cpu_count()} cores",
               "threads": CPU_THREADS_NOTE}
    line = {
        "metric": "preconditioned CGLS iterations/s",
        "value": value,
        "unit": "iter/s",
        "n_gpus": world,
        "steps": K,
        "warmup": Wm,
        "ms_per_step": iter_ms_max / K,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded generators, paper_2603_28642_b200/workloads.py)",
        "config": {
            "workload": name, "mu": args.mu, "p": st["p"], "tau": st["tau"], "coupling": mode,
            "y_mode": pre.y_mode.value, "cg_iters": pre.cg_iters,
            "nnz": {"A": S.nnz, "L1": f.L1.nnz, "L2": f.L2.nnz, "U": f.U.nnz},
            "levels": {"L1": lv_l1[0], "U": lv_u[0], "L1_max_width": lv_l1[1], "U_max_width": lv_u[1]},
            "l2": "flushed (320 MiB write) before every timed iteration, outside the event bracket"
                  if not args.no_flush else "not flushed",
            "parallelism": f"replicas x{world} (one RHS per GPU)",
            "dot_order": (f"exact (reference OpenBLAS association, {args.blas_threads} thread"
                          f"{'s' if args.blas_threads > 1 else ''})"),
        },
        "roofline": {
            "kernel": "triangular solves (+ k_gather_pos), 8 per cg(2) iteration: "
                      + ", ".join(f"{k}: k_trsv_{v[0]}" + (f"<N={v[1]}>" if v[1] else "") for k, v in variants.items()),
            "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "peak_kind": peak_kind, "traffic": traffic,
            "traffic_source": traffic_src,
            "algorithmic_bytes_per_iteration": tbytes, "launches_per_iteration": counts,
            "share_of_step": float(tri_ms[0] / it_ms[0]),
        },
        "cpu_baseline": cpu,
        "e2e": {"value": e2e, "unit": "iter/s", "h2d_bytes_per_step": 8 * S.nrows / K,
                "d2h_bytes_per_step": 8 * S.ncols / K,
                "call": f"pcgls(A, b_pinned_host, pre, CglsConfig(delta=1e-300, max_iters={K})); "
                        "b copied in and x copied out once per call (bytes amortised per iteration)",
                "seconds": e2e_s},
        "gpu_launches": int(K * kpi[0]),
        "clocks": clocks.summary(),
        "rhs_batch": batch,
        "time_to_tol": tol,
        "setup": {**times, "generate_s": t_gen},
        "tri_launches_timed": ntri,
    }
    print(json.dumps(line), flush=True)


def run_rows(args):
    """One RHS, A row-block partitioned across the ranks:
    host-driven iteration with an NCCL allreduce of the n-vector per A^T
    product and an allgather of r for the (replicated) preconditioner apply."""
    import torch
    import torch.distributed as tdist

    import paper_2603_28642_b200 as P
    from paper_2603_28642_b200 import distributed as D

    rank, world, local = dist_env()
    os.environ.setdefault("RSB_DEVICE", str(local))
    torch.cuda.set_device(local)
    tdist.init_process_group("nccl")
    A, b, st, name, _ = make_workload(args, 0)
    S, f, pre, mode, times = setup(args, A, st)
    norm_a = P.power_method_norm2(S, 100, args.config)
    comm = D.TorchComm(device=torch.device("cuda", local))
    mk = lambda Al, pr: D.DeviceBackend(Al, pr, local)  # noqa: E731
    D.pcgls_row_partitioned(S, b, pre, P.CglsConfig(norm_A=norm_a, delta=1e-300, max_iters=args.warmup),
                            comm, mk)
    K = args.steps
    torch.cuda.synchronize()
    tdist.barrier()
    t0 = time.perf_counter()
    _, rep = D.pcgls_row_partitioned(S, b, pre, P.CglsConfig(norm_A=norm_a, delta=1e-300, max_iters=K),
                                     comm, mk)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    t = torch.tensor([dt], dtype=torch.float64, device=f"cuda:{local}")
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    dt = float(t.item())
    if rank == 0:
        print(json.dumps({
            "metric": "preconditioned CGLS iterations/s", "value": rep.iters_run / dt, "unit": "iter/s",
            "n_gpus": world, "steps": K, "warmup": args.warmup, "ms_per_step": 1e3 * dt / max(1, rep.iters_run),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators, paper_2603_28642_b200/workloads.py)",
            "config": {"workload": name, "mu": args.mu, "coupling": mode,
                       "parallelism": f"rows x{world}: A row-partitioned, NCCL allreduce of A^T r, "
                                      "allgather of r, replicated apply",
                       "timing": "wall clock around the fixed-iteration solve, max over ranks"},
        }), flush=True)
    tdist.destroy_process_group()


def main():
    args = parse()
    os.environ["RSB_BLAS_THREADS"] = str(args.blas_threads)
    if args.impl == "reference":
        run_reference(args)
    elif args.partition == "rows" and int(os.environ.get("WORLD_SIZE", "1")) > 1:
        run_rows(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
