"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list as a
markdown table (kernel, launches, mean us, total ms, share).  Usage:
python tools/launch_summary.py launches.csv "title" > profiles/x.md"""
import csv
import sys
from collections import OrderedDict


def main(path, title):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r["Metric Name"] == "gpu__time_duration.sum":
            rows.append((r["Kernel Name"], float(r["Metric Value"].replace(",", "")) / 1e3))
    agg = OrderedDict()
    for k, us in rows:
        name = k.split("(")[0] if k.startswith(("grass", "void grass", "<unnamed>")) else k[:90]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += us
    tot = sum(a[1] for a in agg.values())
    print(f"# {title}\n")
    print(f"{len(rows)} launches, {tot / 1e3:.3f} ms total (serialised, cold-cache per-launch times).\n")
    print("| kernel | launches | mean us | total ms | share |\n|---|---|---|---|---|")
    for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k}` | {n} | {us / n:.1f} | {us / 1e3:.3f} | {100 * us / tot:.1f}% |")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
