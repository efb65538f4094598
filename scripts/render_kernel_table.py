"""Render scripts/kernel_table.py's JSON line as a markdown table.

    python scripts/render_kernel_table.py gpurun_out/.../kernel_table.json > profiles/kernel_table_....md
"""
import json
import sys


def main():
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(f"# Kernel classes alone: {d['config']}")
    print()
    print(f"nnz: {d['nnz']}; HBM peak {d['peak_GBps']} GB/s (MEASURED_PEAKS.json); "
          f"generate {d['generate_s']} s, host ILUP {d['ilup_s']} s.")
    print("Each row: one launch alone, CUDA events on the context stream, L2 flushed before it;")
    print("median of repeats. Algorithmic bytes per SURVEY.md 8(d). Dot rows include the")
    print("host-visible result read (a few microseconds).")
    print()
    print("| kernel | ms | algorithmic MB | GB/s | fraction of peak | notes |")
    print("|---|---|---|---|---|---|")
    for name, r in d["kernels"].items():
        notes = []
        if "levels" in r:
            notes.append(f"{r['levels']} levels (widest {r['max_width']}), {r['us_per_level']} us/level, "
                         f"variant {r['variant']}")
        print(f"| {name} | {r['ms']:.4f} | {r['alg_bytes'] / 1e6:.1f} | {r['GBps']:.0f} | {r['frac']:.3f} | "
              f"{'; '.join(notes)} |")


if __name__ == "__main__":
    main()
