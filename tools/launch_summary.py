"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel:
launches, total and mean duration, share of the library's GPU time."""
import csv
import sys
from collections import defaultdict


def main(path, keep_prefix="spingp_dev::"):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        unit = r["Metric Unit"]
        v = float(r["Metric Value"].replace(",", ""))
        v = v / 1e3 if unit == "ns" else (v if unit == "us" else v * 1e3)
        rows.append((name, v))
    agg = defaultdict(list)
    for n, v in rows:
        if not n.startswith(keep_prefix):  # torch fill/flush, cuBLAS residual checks
            continue
        agg[n].append(v)
    total = sum(sum(v) for v in agg.values())
    print(f"| kernel | launches | total us | mean us | share |\n|---|---|---|---|---|")
    for n, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"| `{n}` | {len(v)} | {sum(v):.1f} | {sum(v) / len(v):.2f} | {100 * sum(v) / total:.1f}% |")
    print(f"\nlibrary kernels: {sum(len(v) for v in agg.values())} launches, {total:.1f} us total "
          f"(library kernels only; torch/cuBLAS kernels of the harness excluded)")


if __name__ == "__main__":
    main(sys.argv[1])
