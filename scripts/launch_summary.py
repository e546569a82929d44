"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per
kernel: launches, average duration, share of the summed GPU time.

  python scripts/launch_summary.py gpurun_out/launches.csv "header line"
"""
import csv
import sys
from collections import defaultdict


def main(path, header=""):
    tot = defaultdict(float)
    cnt = defaultdict(int)
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for row in csv.DictReader(lines):
        if row.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = row["Kernel Name"]
        v = float(row["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3}.get(row["Metric Unit"], 1e-3)
        tot[k] += v * scale
        cnt[k] += 1
    s = sum(tot.values())
    if header:
        print(header)
    print("# per-launch times are cold-cache and serialised; share of the summed GPU time per kernel")
    print(f"{'kernel':72s} {'launches':>9s} {'avg_us':>9s} {'share%':>7s}")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"{k[:72]:72s} {cnt[k]:9d} {tot[k] / cnt[k]:9.2f} {100 * tot[k] / s:7.1f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
