"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per
kernel kind (bench.py's names): launches, total ms, share of the profiled
launches.  ncu serialises launches and runs them cold-cache, so compare the
SHARES with bench.py's kernel_ms_per_step, not the absolute times.

    python tools/launch_summary.py gpurun_out/launches_r01.csv [--out profiles/launches_r01_summary.csv]
"""
import csv
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_traffic import kind  # noqa: E402

TS = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}


def main():
    path = sys.argv[1]
    lines = [ln for ln in open(path) if ln.startswith('"')]
    r = list(csv.reader(lines))
    h = {k: i for i, k in enumerate(r[0])}
    agg = {}
    for row in r[1:]:
        if row[h["Metric Name"]] != "gpu__time_duration.sum":
            continue
        k = kind(row[h["Kernel Name"]])
        ms = float(row[h["Metric Value"]].replace(",", "")) * TS[row[h["Metric Unit"]]]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += ms
    extra = ("validate", "stats")  # bench.py legs outside the timed build
    tot = sum(a[1] for k, a in agg.items() if k not in extra)
    n = sum(a[0] for a in agg.values())
    rows = sorted(agg.items(), key=lambda kv: (kv[0] in extra, -kv[1][1]))
    out = [f"# ncu launch list ({os.path.basename(path)}): {n} launches (cold-cache, serialised; shares only);",
           f"# share = of the {tot:.1f} ms of build kernels; validate/stats = bench.py legs outside the timed build",
           "kernel_kind,launches,total_ms,share"]
    out += [f"{k},{a[0]},{a[1]:.3f},{(a[1] / tot if k not in extra else float('nan')):.4f}" for k, a in rows]
    print("\n".join(out))
    if "--out" in sys.argv:
        open(sys.argv[sys.argv.index("--out") + 1], "w").write("\n".join(out) + "\n")


if __name__ == "__main__":
    main()
