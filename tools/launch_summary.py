"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel launches, total ms and share of GPU time.
usage: python tools/launch_summary.py launches.csv "command" > summary.txt"""
import csv
import sys
from collections import defaultdict


def main():
    path, command = sys.argv[1], sys.argv[2]
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(lines))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        ms = v * {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
                  "nsecond": 1e-6, "second": 1e3}.get(unit, 1e-6)
        k = r["Kernel Name"][:60]
        tot[k] += ms
        cnt[k] += 1
    all_ms = sum(tot.values())
    print("# launch list (ncu --metrics gpu__time_duration.sum --clock-control none; cold-cache, serialised)")
    print(f"# command: {command}")
    print(f"{'kernel':60s} {'launches':>9s} {'total_ms':>10s} {'share':>7s}")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"{k:60s} {cnt[k]:9d} {tot[k]:10.3f} {100 * tot[k] / all_ms:6.2f}%")


if __name__ == "__main__":
    main()
