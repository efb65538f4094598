"""Turn scripts/profile_round.sh outputs (gpurun_out/prof/) into profiles/.

    python scripts/summarize_profiles.py [--round r01]

Writes profiles/launches_<round>_summary.txt (per-iteration kernel shares of
the ncu launch list) and profiles/ncu_trsv_<round>.json (per-launch duration,
DRAM bytes and instruction counts of the triangular solves of one timed
iteration, with their per-iteration sum -- the roofline `traffic` bench.py
reports), and copies the bench lines.
"""
import argparse
import collections
import csv
import json
import os
import shutil

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launches(path):
    rows = []
    with open(path) as fh:
        lines = [l for l in fh if not l.startswith("==")]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            unit = r.get("Metric Unit", "ns")
            v = float(r["Metric Value"].replace(",", ""))
            us = v / 1e3 if unit == "ns" else (v if unit == "us" else v * 1e3)
            rows.append((r["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "").split("::")[-1], us))
    return rows


def iterations(rows):
    """Split at the L2 flush kernel (one before every timed iteration)."""
    its, cur = [], None
    for name, us in rows:
        if name == "k_flush":
            if cur:
                its.append(cur)
            cur = []
            continue
        if cur is not None:
            cur.append((name, us))
    if cur:
        its.append(cur)
    return its


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1, "%": 1}


def raw_rows(path, want):
    with open(path) as fh:
        rd = list(csv.reader(fh))
    hdr, units, data = rd[0], rd[1], rd[2:]
    idx = {w: hdr.index(w) for w in want if w in hdr}
    out = []
    for r in data:
        d = {}
        for w, i in idx.items():
            if w == "Kernel Name":
                d["kernel"] = r[i]
                continue
            try:
                d[w] = float(r[i].replace(",", "")) * SCALE.get(units[i], 1)
            except ValueError:
                pass
        out.append(d)
    return out


def ncu_kernel_table(raw, kt_json, out_path):
    """ncu --set full of every SpMV / wide-solve launch of scripts/kernel_table.py
    (3 launches per row: --reps 1 + 2 warm-up), paired with the event-timed
    table of the same run: DRAM traffic per launch against the algorithmic bytes."""
    kt = json.loads(open(kt_json).read().strip().splitlines()[-1])
    rows = raw_rows(raw, ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                          "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
                          "lts__t_sector_hit_rate.pct"])
    names = [k for k in kt["kernels"] if not k.startswith("dot")]
    lines = [f"# ncu --set full, {kt['config']}",
             "",
             "`ncu --set full --clock-control none -k regex:\"k_spmv|k_trsv_wide\"` on",
             "`python scripts/kernel_table.py --n 2000000 --reps 1`: the last of the 3 launches of each row",
             "(2 warm-up + 1 timed, L2 flushed before each).  Cold-cache and serialised under ncu.",
             "",
             "| row | kernel | ncu us | DRAM MB (read+write) | algorithmic MB | DRAM / algorithmic | warps active % | L2 hit % | regs |",
             "|---|---|---|---|---|---|---|---|---|"]
    per = 3
    for i, name in enumerate(names):
        if (i + 1) * per > len(rows):
            break
        r = rows[(i + 1) * per - 1]
        dram = r.get("dram__bytes_read.sum", 0) + r.get("dram__bytes_write.sum", 0)
        alg = kt["kernels"][name]["alg_bytes"]
        kn = r.get("kernel", "").split("(")[0].replace("void ", "")
        lines.append(f"| {name} | `{kn}` | {1e6 * r.get('gpu__time_duration.sum', 0):.1f} | {dram / 1e6:.1f} | "
                     f"{alg / 1e6:.1f} | {dram / alg:.2f} | "
                     f"{r.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0):.1f} | "
                     f"{r.get('lts__t_sector_hit_rate.pct', 0):.1f} | {r.get('launch__registers_per_thread', 0):.0f} |")
    with open(out_path, "w") as fh:
        fh.write("\n".join(lines) + "\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r01")
    args = ap.parse_args()
    R = args.round
    src = os.path.join(HERE, "gpurun_out", "prof")
    dst = os.path.join(HERE, "profiles")
    for f in (f"bench_{R}.jsonl", f"bench_reference_{R}.jsonl"):
        if os.path.exists(os.path.join(src, f)):
            shutil.copy(os.path.join(src, f), os.path.join(dst, f))
    def launch_summary(csv_name, header, out_name):
        path = os.path.join(src, csv_name)
        if not os.path.exists(path):
            return
        rows = launches(path)
        out = header + [
            "# gpu__time_duration.sum per launch, --clock-control none; serialised and cold-cache under ncu,",
            "# so compare SHARES with bench.py's event-timed numbers, not absolutes.",
            f"# total launches captured: {len(rows)}; each timed iteration follows a k_flush (L2 flush, outside the timed bracket)",
            ""]
        for i, it in enumerate(iterations(rows)):
            tot = sum(us for _, us in it)
            agg = collections.OrderedDict()
            for name, us in it:
                c, t = agg.get(name, (0, 0.0))
                agg[name] = (c + 1, t + us)
            out.append(f"## timed iteration {i}: {len(it)} kernels, {tot:.1f} us summed kernel time")
            for name, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
                out.append(f"  {name:22s} x{c:3d} {t:10.1f} us {100 * t / tot:6.1f}%")
            out.append("")
        with open(os.path.join(dst, out_name), "w") as fh:
            fh.write("\n".join(out))

    launch_summary(f"launches_{R}.csv",
                   [f"# ncu launch list, {R}: `python bench.py --steps 3 --warmup 3 --no-tol --cpu-seconds 1 --batch 0`",
                    "# config 1 (256^2 grid, n=65536, m=98304), ILUP(p=10,tau=0,mu=1), cg(2) coupling solve."],
                   f"launches_{R}_summary.txt")
    launch_summary(f"launches_config4_n2m_{R}.csv",
                   [f"# ncu launch list, {R}: `python bench.py --config 4 --n 2000000 --blas-threads 64 --steps 2 "
                    "--warmup 3 --no-tol --cpu-seconds 1 --batch 0`",
                    "# configs[4] structure at n=2e6 (m=4e6), ILUP(p=10,tau=0,mu=1), cg(2), dots in the 64-thread "
                    "OpenBLAS order."],
                   f"launches_config4_n2m_{R}_summary.txt")
    for f in (f"bench_config4_n8m_{R}.jsonl", f"kernel_table_config4_n8m_{R}.json",
              f"kernel_table_config4_n2m_{R}.json"):
        if os.path.exists(os.path.join(src, f)):
            shutil.copy(os.path.join(src, f), os.path.join(dst, f))
    kt_raw = os.path.join(src, f"kt_{R}.raw.csv")
    kt_json = os.path.join(src, f"kernel_table_config4_n2m_{R}.json")
    if os.path.exists(kt_raw) and os.path.exists(kt_json):
        ncu_kernel_table(kt_raw, kt_json, os.path.join(dst, f"ncu_config4_n2m_{R}.md"))
    raw = os.path.join(src, f"trsv_{R}.raw.csv")
    if os.path.exists(raw):
        with open(raw) as fh:
            rd = list(csv.reader(fh))
        hdr, units, data = rd[0], rd[1], rd[2:]
        want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                "smsp__inst_executed.sum", "sm__cycles_elapsed.max", "launch__registers_per_thread",
                "launch__shared_mem_per_block_dynamic", "launch__shared_mem_per_block_static", "launch__block_size"]
        idx = {w: hdr.index(w) for w in want if w in hdr}
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
                 "msecond": 1e-3, "second": 1}
        launches_ = []
        for r in data:
            d = {}
            for w, i in idx.items():
                v = r[i]
                if w == "Kernel Name":
                    d["kernel"] = v
                    continue
                try:
                    x = float(v.replace(",", ""))
                except ValueError:
                    continue
                u = units[i]
                d[w] = x * scale.get(u, 1)
            launches_.append(d)
        dram = sum(l.get("dram__bytes_read.sum", 0) + l.get("dram__bytes_write.sum", 0) for l in launches_)
        dur = sum(l.get("gpu__time_duration.sum", 0) for l in launches_)
        js = {"source": "ncu --set full --clock-control none -k regex:k_trsv -s 32 -c 8 on python bench.py "
                        "--steps 3 --warmup 3 --no-tol --cpu-seconds 1 --batch 0 (the 8 solves of the first timed "
                        "iteration: 4 L1, 3 L1^T, 1 U; config 1, mu=1)",
              "launches": launches_, "dram_bytes_per_iteration": dram, "duration_s_per_iteration_under_ncu": dur}
        with open(os.path.join(dst, f"ncu_trsv_{R}.json"), "w") as fh:
            json.dump(js, fh, indent=1)
    print("ok")


if __name__ == "__main__":
    main()
