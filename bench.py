"""Benchmark of the B200 solve phase: preconditioned CGLS iterations/s.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config 4 --n N]

Workload (default): BASELINE.json configs[4] at its full size -- n = 8e6,
m = 1.6e7, six nonzeros per row (~96M), rows permuted -- the largest
configuration, and it fits one B200.  Setup follows the reference pipeline
(cli.py:59-94): column_scale, power_method_norm2(100), ilup_factorize(p=10,
tau=0, mu=1), build_preconditioner(cg(2), implicit Y: s = 8e6
exceeds the dense cap), pcgls.  Dots follow the reference's OpenBLAS order
on 64 threads (the order numpy uses on a 64-thread host; the single-thread
order makes every 1.6e7-long dot one serial chain).

A step is one preconditioned CGLS iteration (sv.py:202-241): A p, A^T r, one
row-splitting preconditioner application (8 sparse triangular solves, 3 L2
and 3 L2^T products, the inner-CG dots), the outer dots and the scalar
recursion.  `value` = iterations/s of one right-hand side, device time
(CUDA events on the solver's stream, inputs resident, L2 flushed before
every iteration outside the bracket); `e2e` = the same through the public
pcgls() with b in pinned host memory and x returned; `rhs_batch` = the
8-RHS-per-GPU shard of the 64-RHS batch through pcgls_batch.

--impl reference times the reference's algorithm on the host cores: the
oracle port (oracle/, bit-identical restatement; the reference package is
pure Python and does not exist on the GPU box), set up with the oracle's
own column_scale and ILUP -- no product code is loaded.  Both arms print
the same `config`.  Under torchrun each rank solves its own right-hand
side(s) (replicas, weak scaling); times are the max over ranks.
"""

from __future__ import annotations

import argparse
import hashlib
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
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--mu", type=float, default=1.0)
    ap.add_argument("--mode", default=None, help="coupling solve: dense | cg | identity")
    ap.add_argument("--grid", type=int, default=256, help="config 1 grid side")
    ap.add_argument("--n", type=int, default=None, help="override n (default: the BASELINE size)")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--no-tol", action="store_true", help="skip the time-to-tolerance run")
    ap.add_argument("--no-parity", action="store_true", help="skip the in-run oracle comparison")
    ap.add_argument("--parity-iters", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--batch", type=int, default=8,
                    help="right-hand sides per GPU of the batched solve (0: skip)")
    ap.add_argument("--blas-threads", type=int, default=None,
                    help="reproduce the reference's OpenBLAS dot order at this many threads "
                         "(default: 64 for config 4, else 1)")
    ap.add_argument("--cpu-threads", type=int, default=None,
                    help="host threads of the oracle port (default: all cores)")
    ap.add_argument("--partition", default="replicas", choices=["replicas", "rows"],
                    help="N>1: replicas (RHS per GPU, weak) or rows (one RHS, row-partitioned, strong)")
    a = ap.parse_args()
    if a.blas_threads is None:
        a.blas_threads = 64 if a.config == 4 else 1
    return a


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


# ---------------------------------------------------------------------------
# workload (shared by both arms: numpy generators only)
# ---------------------------------------------------------------------------


def make_workload(args, rank, world):
    """(A, b, B_batch, settings, name, generate_s).  b is this rank's single
    right-hand side; B_batch its shard of the batch."""
    from paper_2603_28642_b200 import workloads as W

    cfgid = args.config
    st = dict(W.SETTINGS[cfgid])
    t0 = time.perf_counter()
    Bb = None
    if cfgid == 4:
        n = args.n or 8_000_000
        nb = max(0, args.batch)
        # rank r: rhs 8r .. 8r+7 of the 64-RHS batch (its shard, rhs_batch);
        # the single-RHS line solves the first of them
        if nb:
            A, Bb = W.config4(seed=4, n=n, nrhs=nb, first_rhs=rank * nb)
            b = Bb[0]
        else:
            A, B1 = W.config4(seed=4, n=n, nrhs=1, first_rhs=rank)
            b = B1[0]
        name = f"config4: random sparse LS, n={A.ncols}, m={A.nrows}, nnz={A.nnz}"
    elif cfgid == 1:
        A, b = W.config1(seed=1, g=args.grid)
        name = f"config1: {args.grid}x{args.grid} grid LS, n={A.ncols}, m={A.nrows}"
    elif cfgid == 0:
        A, b = W.config0(seed=0, **({} if args.n is None else dict(n=args.n, m=3 * args.n // 2)))
        name = f"config0: random sparse LS, n={A.ncols}, m={A.nrows}"
    elif cfgid == 2:
        A, b = W.config2(seed=2, **({} if args.n is None else dict(n=args.n)))
        name = f"config2: sparse + 100 dense rows, n={A.ncols}, m={A.nrows}"
    else:
        A, b = W.config3(seed=3, n=args.n or 1_000_000)
        name = f"config3: ill-conditioned random LS, n={A.ncols}, m={A.nrows}"
    if cfgid != 4:
        if rank > 0:  # replicas: every rank solves its own right-hand side
            b = b + 1e-3 * np.random.default_rng(1000 + rank).standard_normal(len(b))
        if args.batch > 0:
            rng = np.random.default_rng(77 + rank)
            Bb = np.stack([b] + [b + 1e-3 * rng.standard_normal(len(b)) for _ in range(args.batch - 1)])
    return A, np.ascontiguousarray(b), Bb, st, name, time.perf_counter() - t0


def coupling_mode(args, st, s):
    mode = args.mode or st["s_mode"]
    if mode == "dense" and s > 20000:
        mode = "cg"  # the reference CLI's fallback (cli.py:68-78)
    return mode


def config_dict(args, st, name, nnz, mode):
    """The `config` both arms print (identical by construction)."""
    return {
        "workload": name, "mu": args.mu, "p": st["p"], "tau": st["tau"], "coupling": mode,
        "y_mode": "explicit" if mode == "dense" else "implicit", "cg_iters": 2,
        "nnz": nnz, "delta": st["delta"], "max_iters": st["max_iters"],
        "column_scale": bool(st["scale"]),
        "dot_order": (f"reference OpenBLAS ddot association, {args.blas_threads} thread"
                      f"{'s' if args.blas_threads > 1 else ''}"),
        "rhs": "one per pcgls call (sv.py:120); batch shard of 8 per GPU under rhs_batch",
    }


def factor_digest(S_values, f):
    h = hashlib.sha256()
    for a in (S_values, f.row_perm.perm, f.L1.col_ptr, f.L1.row_idx, f.L1.values, f.L2.col_ptr,
              f.L2.row_idx, f.L2.values, f.U.col_ptr, f.U.row_idx, f.U.values):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:16]


def reference_hashes(args, S_values, scale, f):
    """Compare with the digests of the REFERENCE's own setup, when committed
    for this size (tests/golden/cfg4_factor_hashes.json)."""
    if args.config != 4 or args.mu != 1.0:
        return None
    try:
        with open(os.path.join(HERE, "tests", "golden", "cfg4_factor_hashes.json")) as fh:
            want = json.load(fh).get(str(f.U.ncols))
    except OSError:
        return None
    if not want:
        return None
    sys.path.insert(0, os.path.join(HERE, "tests", "golden"))
    from make_cfg4_hashes import factor_digests

    got = factor_digests(S_values, scale, f)
    return all(got[k] == want[k] for k in got)


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
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            time.sleep(0.15)
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


def trsv_bytes_per_iteration(f, mode, cg_iters=2):
    n, s = f.U.ncols, f.L2.nrows
    l1 = tri_bytes(f.L1.nnz, n)
    u = tri_bytes(f.U.nnz, n)
    k = cg_iters
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
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic(workload_key, cls):
    """DRAM bytes (read + write) per iteration of a kernel class ("solves" |
    "products") from the committed ncu capture of this workload
    (scripts/ncu_traffic.py), or (None, why)."""
    path = os.path.join(HERE, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            d = json.load(fh).get(workload_key)
        if d and cls in d:
            per = d[cls].get("per_solve") or d[cls].get("per_product") or {}
            detail = {k: {"dram_bytes": v.get("dram_bytes"), "ncu_ms": v.get("ncu_ms"),
                          "l1tex_pct": v.get("l1tex_pct"), "l2_hit_pct": v.get("l2_hit_pct")} for k, v in per.items()}
            return d[cls].get("dram_bytes_per_iteration"), d[cls].get("source"), detail
    except (OSError, ValueError):
        pass
    return None, "no ncu capture committed for this workload", {}


def spmv_bytes(nnz, rows, cols):
    """int32 indices, f64 values, every operand once."""
    return 12 * nnz + 4 * (rows + 1) + 8 * cols + 8 * rows


def product_bytes_per_iteration(S, f, mode, cg_iters=2):
    """Algorithmic bytes of the sparse products of one iteration: A p, A^T r
    (sv.py:209,234) and the L2 / L2^T products of the apply (pc.py:135-186)."""
    a = spmv_bytes(S.nnz, S.nrows, S.ncols)
    s, n = f.L2.nrows, f.L2.ncols
    l2 = spmv_bytes(f.L2.nnz, s, n)
    if s == 0:
        counts = {"A_x": 1, "AT_y": 1, "L2_t": 0, "L2T_w": 0}
    elif mode == "cg":
        counts = {"A_x": 1, "AT_y": 1, "L2_t": 1 + cg_iters, "L2T_w": 1 + cg_iters}
    elif mode == "identity":
        counts = {"A_x": 1, "AT_y": 1, "L2_t": 1, "L2T_w": 1}
    else:  # dense: the explicit Y takes the place of L2 (its own size is not counted here)
        return 2 * a, {"A_x": 1, "AT_y": 1, "L2_t": 0, "L2T_w": 0}
    return 2 * a + (counts["L2_t"] + counts["L2T_w"]) * l2, counts


def host_cpu():
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        cores = len(os.sched_getaffinity(0))
    except (AttributeError, OSError):
        cores = os.cpu_count()
    return model, cores


# ---------------------------------------------------------------------------
# reference arm: the oracle port on the host cores, no product code
# ---------------------------------------------------------------------------


def oracle_setup(args, A, st):
    from oracle import oracle as O

    t0 = time.perf_counter()
    if st["scale"]:
        S, scale = O.column_scale(A)
    else:
        S, scale = A, np.ones(A.ncols)
    t_scale = time.perf_counter() - t0
    t0 = time.perf_counter()
    f = O.ilup_factorize(S, p=st["p"], tau=st["tau"], mu=args.mu)
    t_ilup = time.perf_counter() - t0
    return S, scale, f, {"column_scale_s": t_scale, "ilup_s": t_ilup}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle as O

    model, cores = host_cpu()
    threads = args.cpu_threads or cores
    O.set_blas_threads(args.blas_threads)
    O.set_cpu_threads(threads)
    A, b, _, st, name, t_gen = make_workload(args, 0, 1)
    S, scale, f, times = oracle_setup(args, A, st)
    mode = coupling_mode(args, st, f.L2.nrows)
    if mode == "dense":
        raise SystemExit("reference arm: dense coupling needs the explicit Y/S build (use --mode cg)")
    t0 = time.perf_counter()
    norm_a = O.power_method_norm2(S, 100, args.config)
    times["power_method_s"] = time.perf_counter() - t0
    op = O.OraclePreconditioner(f, mode, "implicit", 2)
    O.pcgls(S, b, op, norm_a, delta=1e-300, max_iters=max(1, args.warmup))
    k = args.steps
    t0 = time.perf_counter()
    _, rep = O.pcgls(S, b, op, norm_a, delta=1e-300, max_iters=k)
    dt = time.perf_counter() - t0
    value = k / dt
    # the reference's time to tolerance on the host: power method + pcgls to delta
    t0 = time.perf_counter()
    _, rtol = O.pcgls(S, b, op, norm_a, delta=st["delta"], max_iters=st["max_iters"])
    t_solve = time.perf_counter() - t0
    tol = {"seconds": times["power_method_s"] + t_solve, "power_method_s": times["power_method_s"],
           "solve_s": t_solve, "its": rtol["its"], "converged": rtol["converged"], "delta": st["delta"],
           "includes": "power method (100 its) + pcgls to delta on the host cores; ILUP in `setup`"}
    nnz = {"A": S.nnz, "L1": f.L1.nnz, "L2": f.L2.nnz, "U": f.U.nnz}
    sample = (f"{k} fixed iterations (delta=1e-300) of the oracle port of pcgls on this config "
              f"after {args.warmup} warm-up iterations")
    line = {
        "impl": "reference", "metric": "preconditioned CGLS iterations/s", "value": value,
        "unit": "iter/s", "n_gpus": args.gpus, "steps": k, "warmup": args.warmup,
        "ms_per_step": 1e3 * dt / k, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded generators, paper_2603_28642_b200/workloads.py)",
        "config": config_dict(args, st, name, nnz, mode),
        "cpu_baseline": {"value": value, "unit": "iter/s", "cores": threads, "kind": "port",
                         "sample": sample, "host_cpu": model, "host_cores": cores},
        "e2e": {"value": value, "unit": "iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "time_to_tol": tol,
        "setup": {**times, "generate_s": t_gen, "factor_digest": factor_digest(S.values, f)},
        "native_libs": loaded_native_libs(),
    }
    print(json.dumps(line), flush=True)


def loaded_native_libs():
    try:
        with open("/proc/self/maps") as fh:
            libs = {ln.split()[-1] for ln in fh if ln.rstrip().endswith(".so") and HERE in ln}
        return sorted(os.path.relpath(p, HERE) for p in libs)
    except OSError:
        return None


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------


def product_setup(args, A, st):
    import paper_2603_28642_b200 as P

    times = {}
    t0 = time.perf_counter()
    if st["scale"]:
        S, sc = P.column_scale(A)
        scale = sc.scale
    else:
        S, scale = A, np.ones(A.ncols)
    times["column_scale_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    from paper_2603_28642_b200.ilup import ilup_factorize_cached

    f = ilup_factorize_cached(S, P.IlupParams(p=st["p"], tau=st["tau"], mu=args.mu))  # $RSB_FACTOR_CACHE
    times["ilup_host_s"] = time.perf_counter() - t0
    times["ilup_cache"] = os.environ.get("RSB_FACTOR_CACHE") is not None
    mode = coupling_mode(args, st, f.L2.nrows)
    t0 = time.perf_counter()
    pre = P.build_preconditioner(f, s_mode=P.SMode(mode))
    times["build_preconditioner_s"] = time.perf_counter() - t0
    return S, scale, f, pre, mode, times


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
    from paper_2603_28642_b200 import device as D

    A, b, Bb, st, name, t_gen = make_workload(args, rank, world)
    S, scale, f, pre, mode, times = product_setup(args, A, st)
    ctx = D.get_context()
    t0 = time.perf_counter()
    dA = D.device_matrix(S, ctx)
    dpre = D.device_preconditioner(pre, ctx)
    solver = D.device_solver(dA, dpre)
    ctx.sync()
    times["upload_and_analysis_s"] = time.perf_counter() - t0
    lv_l1 = dpre.L1.levels(L.TRI_LOWER_UNIT)
    lv_u = dpre.U.levels(L.TRI_UPPER)
    variants = {"L1": dpre.L1.variant(L.TRI_LOWER_UNIT), "U": dpre.U.variant(L.TRI_UPPER)}
    if f.L2.nrows:
        variants["L1T"] = dpre.L1.variant(L.TRI_LOWER_T_UNIT)
    t0 = time.perf_counter()
    norm_a = P.power_method_norm2(S, 100, args.config)
    times["power_method_device_s"] = time.perf_counter() - t0

    K, Wm = args.steps, args.warmup
    # ---- device-resident timed region: K iterations as graph replays
    bdev = D.DeviceBuffer(ctx, len(b))
    bdev.upload(b)
    cfg = solver.cfg_struct(norm_a, 1e-300, Wm + K + 8, 5, False)
    status = solver.start(bdev.ptr, L.RSB_DEVICE, cfg)
    if status != 0:
        raise RuntimeError(f"solver stopped at start (status {status})")
    solver.iterate(Wm)
    it_ms, tri_ms = np.zeros(1), np.zeros(1)
    tri_launches, kpi = np.zeros(1, dtype=np.int64), np.zeros(1, dtype=np.int64)
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
    prod_ms, prod_launches = np.zeros(1), np.zeros(1, dtype=np.int64)
    L.check(L.lib().rsb_solver_bench_products(solver.h, prod_ms.ctypes.data_as(L.f64p),
                                              prod_launches.ctypes.data_as(L.i64p)))

    # ---- end to end through the public API (host buffers, copies inside)
    bpin = D.PinnedBuffer(len(b))
    bpin.array[:] = b
    e2e_cfg = P.CglsConfig(norm_A=norm_a, delta=1e-300, max_iters=K)
    P.pcgls(S, bpin.array, pre, P.CglsConfig(norm_A=norm_a, delta=1e-300, max_iters=max(1, Wm)))
    barrier()
    t0 = time.perf_counter()
    x_e2e, rep = P.pcgls(S, bpin.array, pre, e2e_cfg)
    e2e_s = barrier_max(time.perf_counter() - t0)
    e2e = world * K / e2e_s

    # ---- the batch shard of right-hand sides per GPU
    batch = None
    if Bb is not None and len(Bb) > 1:
        # the shard's right-hand sides in page-locked host memory, as b above
        Bpin = D.PinnedBuffer(Bb.size)
        Bp = Bpin.array.reshape(Bb.shape)
        Bp[:] = Bb
        P.pcgls_batch(S, Bp, pre, P.CglsConfig(norm_A=norm_a, delta=1e-300, max_iters=max(1, Wm)))
        barrier()
        t0 = time.perf_counter()
        _, breps = P.pcgls_batch(S, Bp, pre, e2e_cfg)
        b_s = barrier_max(time.perf_counter() - t0)
        its = sum(K if r.converged else r.its for r in breps)
        # device-resident: the batched iteration graph replayed K times
        dev = None
        bsv = D.device_batch_solver(D.device_matrix(S, ctx), D.device_preconditioner(pre, ctx))
        if bsv is not None and len(Bb) <= D.BATCH:
            bst = bsv.start(np.ascontiguousarray(Bb), solver.cfg_struct(norm_a, 1e-300, Wm + K + 8, 5, False))
            if all(v == 0 for v in bst):
                bsv.iterate(Wm)
                bit, btri = np.zeros(1), np.zeros(1)
                btl, bkpi = np.zeros(1, dtype=np.int64), np.zeros(1, dtype=np.int64)
                bdone = L.ctypes.c_int()
                barrier()
                L.check(L.lib().rsb_bsolver_bench(bsv.h, K, 0 if args.no_flush else 1, bit.ctypes.data_as(L.f64p),
                                                  btri.ctypes.data_as(L.f64p), btl.ctypes.data_as(L.i64p),
                                                  bkpi.ctypes.data_as(L.i64p), L.ctypes.byref(bdone)))
                bms = barrier_max(float(bit[0]))
                dev = {"value": world * len(Bb) * K / (bms / 1e3), "unit": "RHS-iter/s",
                       "ms_per_iteration": bms / K, "trsv_share": float(btri[0] / bit[0]),
                       "kernels_per_iteration": int(bkpi[0]),
                       "timing": "CUDA events around K replays of the batch's iteration graph, inputs resident"}
        batch = {"rhs_per_gpu": len(Bb), "value": world * its / b_s, "unit": "RHS-iter/s",
                 "seconds": b_s, "its_each": K, "device": dev,
                 "path": "batched kernels (csrc/bsolver.cu)" if bsv is not None else "one stream per RHS",
                 "call": f"pcgls_batch(A, B[{len(Bb)} x m] pinned host, pre, CglsConfig(delta=1e-300, "
                         f"max_iters={K})), H2D of B and D2H of X inside"}

    # ---- time to tolerance: power method + upload + level analysis + solve
    tol = None
    if not args.no_tol:
        D.clear_caches()
        dA = dpre = solver = None
        t0 = time.perf_counter()
        D.device_matrix(S, ctx)
        D.device_preconditioner(pre, ctx)
        ctx.sync()
        t_up = time.perf_counter() - t0
        nrm = P.power_method_norm2(S, 100, args.config)
        t_pm = time.perf_counter() - t0 - t_up
        x_tol, rtol = P.pcgls(S, b, pre, P.CglsConfig(norm_A=nrm, delta=st["delta"], max_iters=st["max_iters"]))
        t_all = barrier_max(time.perf_counter() - t0)
        tol = {"seconds": t_all, "upload_and_analysis_s": t_up, "power_method_s": t_pm,
               "solve_s": t_all - t_up - t_pm, "its": rtol.its,
               "converged": rtol.converged, "breakdown": rtol.breakdown, "delta": st["delta"],
               "ratio_pt_final": rtol.ratio_pt_final,
               "grad_ratio": rtol.gradient_norm_final / (nrm * rtol.residual_norm_final)
               if rtol.residual_norm_final > 0 else 0.0,
               "includes": "upload + triangular-solve level analysis + power method (100 its) + pcgls "
                           "to delta with host b in / x out; ILUP and build are in `setup`"}

    if rank != 0:
        if dist is not None:
            dist[1].destroy_process_group()
        return
    # ---- roofline of the dominant kernel class: the triangular solves or the
    # sparse products, whichever took more of the timed iterations (both
    # classes are reported; event pairs around every launch of the class)
    peak, peak_kind = measured_peak()
    wkey = f"config{args.config}_n{S.ncols}_mu{args.mu}_{mode}"
    tbytes, counts = trsv_bytes_per_iteration(f, mode)
    pbytes, pcounts = product_bytes_per_iteration(S, f, mode)
    classes = {}
    for cls, label, by, cnt, ms in (
            ("solves", "sparse triangular solves", tbytes, counts, float(tri_ms[0])),
            ("products", "sparse products (A x, A^T y, L2 t, L2^T w)", pbytes, pcounts, float(prod_ms[0]))):
        tr, tr_src, tr_detail = ncu_traffic(wkey, cls)
        ach = (by * K) / (ms / 1e3) / 1e9 if ms > 0 else 0.0
        classes[cls] = {"kernel": f"{label}, {sum(cnt.values())} per iteration ({cnt})", "bound": "hbm",
                        "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak, "peak_kind": peak_kind,
                        "traffic": tr, "traffic_source": tr_src, "ncu_per_kernel": tr_detail,
                        "algorithmic_bytes_per_iteration": by,
                        "ms_per_iteration": ms / K, "share_of_step": ms / float(it_ms[0])}
    dom = max(classes, key=lambda c: classes[c]["ms_per_iteration"])
    roofline = dict(classes[dom])
    roofline["other_class"] = {c: v for c, v in classes.items() if c != dom}
    roofline["note"] = ("classes overlap in time: A^T r runs on a side branch concurrently with the preconditioner "
                        "application, so the shares can sum past 1; random 8-byte gathers are bounded by the L1TEX "
                        "wavefront rate, not by HBM (DESIGN.md section 5)")
    model, cores = host_cpu()

    # ---- parity against the oracle port + the CPU baseline (rank 0, N = 1)
    parity, cpu = None, None
    if world == 1 and not args.no_parity and mode != "dense":
        from oracle import oracle as O

        threads = args.cpu_threads or max(1, cores - 1)
        O.set_blas_threads(args.blas_threads)
        O.set_cpu_threads(threads)
        t0 = time.perf_counter()
        norm_o = O.power_method_norm2(S, 100, args.config)
        t_pm_o = time.perf_counter() - t0
        op = O.OraclePreconditioner(f, mode, "implicit", 2)
        kp = max(1, args.parity_iters)
        t0 = time.perf_counter()
        xo, ro = O.pcgls(S, b, op, norm_o, delta=1e-300, max_iters=kp)
        t_o = time.perf_counter() - t0
        xg, rg = P.pcgls(S, b, pre, P.CglsConfig(norm_A=norm_a, delta=1e-300, max_iters=kp))
        ro["psize"] = pre.psize  # the oracle preconditioner carries no Y / S factor to count
        rd = rg.to_dict()
        parity = {"iters": kp, "norm_A_bitwise": norm_a == norm_o, "x_bitwise": bool(np.array_equal(xg, xo)),
                  "report_equal": rd == ro,
                  "report_diff": sorted(k for k in rd if rd.get(k) != ro.get(k)),
                  "factors_match_reference_hashes": reference_hashes(args, S.values, scale, f),
                  "factor_digest": factor_digest(S.values, f),
                  "checker": "oracle port (oracle/), same scaled A, factors and b; fixed-iteration pcgls"}
        # CPU baseline: a bounded sample of the same workload on the host cores
        rate = kp / t_o
        if t_o < args.cpu_seconds:
            kc = int(max(kp, min(400, args.cpu_seconds / max(t_o / kp, 1e-4))))
            t0 = time.perf_counter()
            O.pcgls(S, b, op, norm_o, delta=1e-300, max_iters=kc)
            t_o, kp = time.perf_counter() - t0, kc
            rate = kc / t_o
        cpu = {"value": rate, "unit": "iter/s", "cores": threads, "kind": "port",
               "sample": f"{kp} fixed iterations (delta=1e-300) of the oracle port of pcgls on this config, "
                         f"{t_o:.1f} s (power method {t_pm_o:.1f} s not included)",
               "host_cpu": model, "host_cores": cores}

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
        "config": config_dict(args, st, name, {"A": S.nnz, "L1": f.L1.nnz, "L2": f.L2.nnz, "U": f.U.nnz}, mode),
        "device": {
            "levels": {"L1": lv_l1[0], "U": lv_u[0], "L1_max_width": lv_l1[1], "U_max_width": lv_u[1]},
            "trsv_kernels": {k: v[0] + (f"<N={v[1]}>" if v[1] else "") for k, v in variants.items()},
            "l2": "flushed (320 MiB write) before every timed iteration, outside the event bracket"
                  if not args.no_flush else "not flushed",
            "parallelism": f"replicas x{world}",
        },
        "roofline": roofline,
        "cpu_baseline": cpu,
        "parity": parity,
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
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist[1].destroy_process_group()


def run_rows(args):
    """One RHS, A's rows (and L2's with them) partitioned across the ranks
    (SURVEY.md 8(e)): distributed.py's loop on the device backend, NCCL
    collectives on the library's stream; strong scaling."""
    import torch
    import torch.distributed as tdist

    import paper_2603_28642_b200 as P
    from paper_2603_28642_b200 import distributed as DI

    for k, v in (("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29517"), ("RANK", "0"), ("WORLD_SIZE", "1"),
                 ("LOCAL_RANK", "0")):
        os.environ.setdefault(k, v)  # a single-process run without torchrun
    rank, world, local = dist_env()
    os.environ.setdefault("RSB_DEVICE", str(local))
    torch.cuda.set_device(local)
    tdist.init_process_group("nccl")
    args.batch = 0
    A, b, _, st, name, _ = make_workload(args, 0, 1)
    S, scale, f, pre, mode, times = product_setup(args, A, st)
    norm_a = P.power_method_norm2(S, 100, args.config)
    comm = DI.TorchComm(device=torch.device("cuda", local), reduce=os.environ.get("RSB_ROWS_REDUCE", "ordered"))
    be = DI.DeviceBackend(local)
    with be.stream_context():
        part = DI.RowPartition(S, pre, comm, be)  # uploads + analyses, outside the timed region
    DI.pcgls_row_partitioned(S, b, pre, P.CglsConfig(norm_A=norm_a, delta=1e-300, max_iters=max(1, args.warmup)),
                             comm, be, part)
    K = args.steps
    torch.cuda.synchronize()
    tdist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(be.stream)
    _, rep = DI.pcgls_row_partitioned(S, b, pre, P.CglsConfig(norm_A=norm_a, delta=1e-300, max_iters=K), comm, be,
                                      part)
    ev1.record(be.stream)
    torch.cuda.synchronize()
    dt = ev0.elapsed_time(ev1) / 1e3
    t = torch.tensor([dt], dtype=torch.float64, device=f"cuda:{local}")
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    dt = float(t.item())
    if rank == 0:
        print(json.dumps({
            "metric": "preconditioned CGLS iterations/s", "value": rep.iters_run / dt, "unit": "iter/s",
            "n_gpus": world, "steps": K, "warmup": args.warmup, "ms_per_step": 1e3 * dt / max(1, rep.iters_run),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators, paper_2603_28642_b200/workloads.py)",
            "config": config_dict(args, st, name, {"A": S.nnz, "L1": f.L1.nnz, "L2": f.L2.nnz, "U": f.U.nnz},
                                  mode),
            "parallelism": f"rows x{world}: A and L2 row blocks, replicated L1/U solves, "
                           f"{comm.reduce} sums of the A^T / L2^T partials",
            "timing": "CUDA events on the library stream around the fixed-iteration solve (includes the "
                      "host's control flow), max over ranks",
        }), flush=True)
    tdist.destroy_process_group()


def main():
    args = parse()
    os.environ["RSB_BLAS_THREADS"] = str(args.blas_threads)
    if args.impl == "reference":
        run_reference(args)
    elif args.partition == "rows":
        run_rows(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
