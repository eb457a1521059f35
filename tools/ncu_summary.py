"""One-screen summary of ncu --set full reports: duration, DRAM, tensor pipe,
issue rate, busiest pipes, top stall instructions.
    python tools/ncu_summary.py report1.ncu-rep [report2 ...]"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.per_cycle_active", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2]


def main():
    for rep in sys.argv[1:]:
        h, u, v = raw(rep)
        print(f"== {rep}")
        print("  kernel:", v[h.index("Kernel Name")][:110])
        for k in KEYS:
            if k in h:
                print(f"  {k:70s} {v[h.index(k)]:>14s} {u[h.index(k)]}")
        pipes = []
        for i, k in enumerate(h):
            if k.startswith("sm__inst_executed_pipe_") and k.endswith(".avg.pct_of_peak_sustained_active"):
                try:
                    if float(v[i]) > 5:
                        pipes.append((float(v[i]), k.split("pipe_")[1].split(".")[0]))
                except ValueError:
                    pass
        print("  pipes (% of peak, active):", ", ".join(f"{n} {p:.0f}" for p, n in sorted(pipes, reverse=True)))


if __name__ == "__main__":
    main()
