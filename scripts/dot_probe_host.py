"""Dot-association probe on THIS host's CPU.

    python scripts/dot_probe_host.py [--threads 1,2,4,8,16] [--write-golden]

For each OpenBLAS thread count T (one subprocess each: OpenBLAS reads
OPENBLAS_NUM_THREADS at load time and caps it at the core count) the child
computes numpy's `a @ b` on seeded vectors of the lengths of
tests/golden/make_golden_mt.py and compares every result bit for bit with
the oracle's restatement of the OpenBLAS association (oracle.set_blas_threads(T);
oracle/rsref.c).  Prints one JSON line: CPU model, cores, numpy / OpenBLAS
versions, per-T match.  --write-golden adds the numpy results to
tests/golden/dots_mt_host.json (fixtures for T above this container's 8 cores).
"""
import argparse
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DOT_LENS = [10000, 10001, 10002, 16384, 20001, 33333, 65536, 98304, 131071, 262147, 1000003, 8000000, 16000000]
SEED = 4242


def child(t):
    import numpy as np

    sys.path.insert(0, HERE)
    from oracle import oracle as O

    O.set_blas_threads(t)
    rng = np.random.default_rng(SEED)
    vals, same = [], []
    for n in DOT_LENS:
        a, b = rng.standard_normal(n), rng.standard_normal(n)
        v = float(a @ b)
        vals.append(v)
        same.append(bool(v == O.dot(a, b)))
    info = {}
    try:
        from threadpoolctl import threadpool_info

        info = [{k: d.get(k) for k in ("internal_api", "version", "num_threads", "architecture")}
                for d in threadpool_info()]
    except Exception:  # noqa: BLE001
        pass
    print(json.dumps({"vals": vals, "same": same, "blas": info}))


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", default="1,2,4,8,16")
    ap.add_argument("--write-golden", action="store_true")
    ap.add_argument("--child", type=int, default=0)
    args = ap.parse_args()
    if args.child:
        child(args.child)
        return
    import numpy as np

    out = {"host_cpu": cpu_model(), "cores": os.cpu_count(), "numpy": np.__version__, "lens": DOT_LENS, "seed": SEED,
           "threads": {}}
    golden = {"lens": DOT_LENS, "seed": SEED, "host_cpu": out["host_cpu"], "cores": out["cores"], "dots": {}}
    for t in [int(v) for v in args.threads.split(",")]:
        if t > (os.cpu_count() or 1):
            out["threads"][str(t)] = "skipped: more threads than cores (OpenBLAS caps at the core count)"
            continue
        env = dict(os.environ, OPENBLAS_NUM_THREADS=str(t))
        r = subprocess.run([sys.executable, __file__, "--child", str(t)], env=env, check=True, capture_output=True,
                           text=True)
        d = json.loads(r.stdout.strip().splitlines()[-1])
        out["threads"][str(t)] = {"all_bitwise_equal_to_oracle": all(d["same"]), "same": d["same"], "blas": d["blas"]}
        golden["dots"][str(t)] = d["vals"]
    if args.write_golden:
        with open(os.path.join(HERE, "tests", "golden", "dots_mt_host.json"), "w") as fh:
            json.dump(golden, fh, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
