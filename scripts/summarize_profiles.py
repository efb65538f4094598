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
    rows = launches(os.path.join(src, f"launches_{R}.csv"))
    out = [f"# ncu launch list, {R}: `python bench.py --steps 3 --warmup 3 --no-tol --cpu-seconds 1 --batch 0`",
           "# config 1 (256^2 grid, n=65536, m=98304), ILUP(p=10,tau=0,mu=1), cg(2) coupling solve.",
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
    with open(os.path.join(dst, f"launches_{R}_summary.txt"), "w") as fh:
        fh.write("\n".join(out))
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
