"""profiles/ncu_traffic.json from two `ncu --set full` raw CSV exports at
configs[4] full size (the bench's `roofline.traffic`):

    ncu --set full --clock-control none -k regex:"k_trsv|k_wide|k_fill" -o trsv python scripts/trsv_once.py --n 8000000
    ncu --set full --clock-control none -k regex:"k_spmv" -o spmv python scripts/kernel_table.py --n 8000000 --reps 1
    ncu -i trsv.ncu-rep --page raw --csv > trsv.raw.csv ; ncu -i spmv.ncu-rep --page raw --csv > spmv.raw.csv
    python scripts/ncu_traffic.py --trsv trsv.raw.csv --spmv spmv.raw.csv --n 8000000

Solves: the LAST launch of each solve kernel kind (mode 0 = L1, 1 = L1^T, 2 = U)
plus the sentinel fill before it.  Products: the last launch of each product
in kernel_table.py's order (A x, A^T y, L2 t, L2^T w).  Per iteration of the
cg(2) apply: 4 L1 + 3 L1^T + 1 U solves; A x + A^T y + 3 L2 t + 3 L2^T w.
"""
import argparse
import csv
import json
import os
import re

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rows_of(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}

    def val(r, name):
        v = float(r[idx[name]].replace(",", ""))
        u = units[idx[name]].lower()
        scale = {"gbyte": 1e9, "mbyte": 1e6, "kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "us": 1e-6, "ns": 1e-9,
                 "msecond": 1e-3, "usecond": 1e-6, "nsecond": 1e-9, "second": 1.0}.get(u, 1.0)
        return v * scale

    out = []
    for r in rows[2:]:
        out.append({"name": r[idx["Kernel Name"]],
                    "dram": val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum"),
                    "sec": val(r, "gpu__time_duration.sum"),
                    "l2_hit": float(r[idx["lts__t_sector_hit_rate.pct"]]),
                    "l1tex_pct": float(r[idx["l1tex__throughput.avg.pct_of_peak_sustained_elapsed"]])
                    if "l1tex__throughput.avg.pct_of_peak_sustained_elapsed" in idx else None})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trsv", required=True)
    ap.add_argument("--spmv", required=True)
    ap.add_argument("--n", type=int, default=8_000_000)
    ap.add_argument("--key", default=None)
    ap.add_argument("--out", default=os.path.join(HERE, "profiles", "ncu_traffic.json"))
    args = ap.parse_args()
    key = args.key or f"config4_n{args.n}_mu1.0_cg"
    tr = rows_of(args.trsv)
    solve = {}
    fill = [r for r in tr if "k_fill" in r["name"]]
    for r in tr:
        m = re.search(r"k_trsv_\w+<\(?(?:int\))?(\d)", r["name"])
        if m:
            solve[{"0": "L1", "1": "L1T", "2": "U", "3": "U"}[m.group(1)]] = r  # the last launch wins
    fill_b = fill[-1]["dram"] if fill else 0.0
    fill_s = fill[-1]["sec"] if fill else 0.0
    per_solve = {k: {"dram_bytes": v["dram"] + fill_b, "ncu_ms": (v["sec"] + fill_s) * 1e3, "l2_hit_pct": v["l2_hit"],
                     "l1tex_pct": v["l1tex_pct"], "kernel": v["name"][:60]} for k, v in solve.items()}
    counts = {"L1": 4, "L1T": 3, "U": 1}
    solves_iter = sum(counts[k] * per_solve[k]["dram_bytes"] for k in counts)
    sp = [r for r in rows_of(args.spmv) if "k_spmv" in r["name"]]
    names = ["A_x", "AT_y", "L2_t", "L2T_w"]
    per = len(sp) // 4
    prod = {}
    for i, nm in enumerate(names):
        r = sp[(i + 1) * per - 1]
        prod[nm] = {"dram_bytes": r["dram"], "ncu_ms": r["sec"] * 1e3, "l2_hit_pct": r["l2_hit"],
                    "l1tex_pct": r["l1tex_pct"], "kernel": r["name"][:60]}
    pc = {"A_x": 1, "AT_y": 1, "L2_t": 3, "L2T_w": 3}
    prod_iter = sum(pc[k] * prod[k]["dram_bytes"] for k in pc)
    path = args.out
    try:
        allk = json.load(open(os.path.join(HERE, "profiles", "ncu_traffic.json")))
    except (OSError, ValueError):
        allk = {}
    allk[key] = {
        "solves": {"dram_bytes_per_iteration": solves_iter, "per_solve": per_solve, "counts": counts,
                   "source": "ncu --set full --clock-control none of scripts/trsv_once.py --n %d (sentinel fill + solve kernel, "
                             "second run of each); per iteration = 4 L1 + 3 L1^T + 1 U" % args.n},
        "products": {"dram_bytes_per_iteration": prod_iter, "per_product": prod, "counts": pc,
                     "source": "ncu --set full --clock-control none of scripts/kernel_table.py --n %d --reps 1 (last launch of "
                               "each product); per iteration = A x + A^T y + 3 L2 t + 3 L2^T w" % args.n},
    }
    json.dump(allk, open(path, "w"), indent=1)
    print(json.dumps(allk[key], indent=1))


if __name__ == "__main__":
    main()
