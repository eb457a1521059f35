"""Per-launch DRAM throughput from an ncu CSV with gpu__time_duration.sum,
dram__bytes_read.sum, dram__bytes_write.sum:
    python tools/launch_bw.py launches.csv [kernel-substring]"""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Metric Name" in r][0]
    h = rows[hi]
    K, M, V, ID = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    U = h.index("Metric Unit")
    d = collections.OrderedDict()
    for r in rows[hi + 1:]:
        v = float(r[V].replace(",", ""))
        unit = r[U]
        if unit in ("nsecond", "ns"):
            v *= 1e-9
        elif unit in ("usecond", "us"):
            v *= 1e-6
        elif unit in ("msecond", "ms"):
            v *= 1e-3
        elif unit == "Kbyte":
            v *= 1e3
        elif unit == "Mbyte":
            v *= 1e6
        elif unit == "Gbyte":
            v *= 1e9
        d.setdefault((int(r[ID]), r[K]), {})[r[M]] = v
    return d


def main():
    d = load(sys.argv[1])
    sub = sys.argv[2] if len(sys.argv) > 2 else None
    agg = collections.defaultdict(lambda: [0.0, 0.0, 0])
    for (i, k), m in d.items():
        t = m.get("gpu__time_duration.sum", 0.0)
        b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        name = k.split("(")[0]
        if sub:
            if sub in name:
                print(f"{i:5d} {t * 1e6:9.1f} us {b / 1e6:9.1f} MB {b / t / 1e12 if t else 0:6.2f} TB/s  {name[:60]}")
            continue
        a = agg[name]
        a[0] += t
        a[1] += b
        a[2] += 1
    for name, (t, b, n) in sorted(agg.items(), key=lambda x: -x[1][0])[:30]:
        print(f"{t * 1e3:8.3f} ms {b / 1e9:7.2f} GB {b / t / 1e12:5.2f} TB/s n={n:3d} {name[:70]}")


if __name__ == "__main__":
    main()
