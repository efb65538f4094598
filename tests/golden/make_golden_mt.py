"""Golden fixtures of the REFERENCE run with a multi-threaded OpenBLAS.

    python tests/golden/make_golden_mt.py          (needs >= 8 cores)

numpy's OpenBLAS splits a dot longer than 10000 over
min(OPENBLAS_NUM_THREADS, cores) threads, which changes its bits
(SURVEY.md Appendix B).  The product's RSB_BLAS_THREADS=T order and the
oracle's set_blas_threads(T) reproduce that split; these fixtures pin both
against the reference itself:

  dots_mt.json     `a @ b` at T = 2, 4, 8 threads on seeded vectors
                   (one subprocess per T, since OpenBLAS reads the variable
                   at load time)
  cfg1m_t8.npz/    the reference pipeline (column_scale, power method, ILUP,
  _reports.json    build_preconditioner, pcgls) on configs[1] at a 112^2 grid
                   (n = 12,544 > 10000: every n- and m-long dot and norm is
                   threaded) with OPENBLAS_NUM_THREADS = 8
"""

from __future__ import annotations

import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
DOT_LENS = [10000, 10001, 10002, 16384, 20001, 33333, 65536, 98304, 131071, 262147, 1000003]


def dots_child(t):
    import numpy as np

    rng = np.random.default_rng(4242)
    vals = []
    for n in DOT_LENS:
        a, b = rng.standard_normal(n), rng.standard_normal(n)
        vals.append(float(a @ b))
    print(json.dumps(vals))


def solve_child():
    sys.argv = [sys.argv[0]]
    sys.path.insert(0, HERE)
    import make_golden as G  # noqa: E402  (imports the reference; env already set)

    A, b = G.W.config1(seed=1, g=112)
    G.solve_fixture("cfg1m_t8", A, b, dict(p=10, tau=0.0, mu=1.0), ["cg", "identity"], 1e-10, 25, rs_seed=1)


def main():
    if os.cpu_count() < 8:
        sys.exit("needs >= 8 cores (OpenBLAS caps its threads at the core count)")
    out = {"lens": DOT_LENS, "seed": 4242, "dots": {}}
    for t in (2, 4, 8):
        env = dict(os.environ, OPENBLAS_NUM_THREADS=str(t))
        r = subprocess.run([sys.executable, __file__, "--dots", str(t)], env=env, check=True,
                           capture_output=True, text=True)
        out["dots"][str(t)] = json.loads(r.stdout)
    with open(os.path.join(HERE, "dots_mt.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    env = dict(os.environ, OPENBLAS_NUM_THREADS="8")
    subprocess.run([sys.executable, __file__, "--solve"], env=env, check=True)
    print("multi-thread fixtures written to", HERE)


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--dots":
        dots_child(int(sys.argv[2]))
    elif len(sys.argv) > 1 and sys.argv[1] == "--solve":
        solve_child()
    else:
        main()
