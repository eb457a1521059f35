"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel name."""
import csv
import sys
from collections import defaultdict


def main(path, top=40):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rd = csv.DictReader(lines)
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        v = v / 1e6 if unit in ("nsecond", "ns") else (v / 1e3 if unit in ("usecond", "us") else v)
        tot[name[:110]] += v
        cnt[name[:110]] += 1
    T = sum(tot.values())
    print(f"total {T:.2f} ms over {sum(cnt.values())} launches")
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:top]:
        print(f"{v:8.3f} ms {100*v/T:5.1f}% {cnt[k]:5d}  {k}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
