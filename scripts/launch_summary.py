"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per kernel family, launches, ms per launch and share of the total."""
import collections
import csv
import sys


def main(path, top=20):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        v = float(d["Metric Value"]) * {"usecond": 1e3, "msecond": 1e6}.get(d["Metric Unit"], 1)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{k[-48:]:48s} {v[0]:5d} {v[1] / 1e6 / v[0]:9.4f} ms/launch {100 * v[1] / tot:5.1f}%")
    print(f"total {tot / 1e6:.3f} ms over {sum(v[0] for v in agg.values())} launches")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 20)
