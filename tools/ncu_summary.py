"""Summarise an ncu report: per-launch time, DRAM bytes, achieved GB/s, occupancy.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--csv out.csv]
"""
import csv
import subprocess
import sys

METS = ("gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
        "sm__warps_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed,"
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed,"
        "launch__registers_per_thread,lts__t_sectors.sum")
TS = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
BS = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", METS],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, units = r[0], r[1]
    idx = {k: i for i, k in enumerate(h)}

    def num(row, k, table):
        return float(row[idx[k]].replace(",", "")) * table[units[idx[k]]]

    for row in r[2:]:
        yield {
            "kernel": row[idx["Kernel Name"]],
            "time_us": num(row, "gpu__time_duration.sum", TS),
            "dram_read_MB": num(row, "dram__bytes_read.sum", BS),
            "dram_write_MB": num(row, "dram__bytes_write.sum", BS),
            "l2_MB": float(row[idx["lts__t_sectors.sum"]].replace(",", "")) * 32e-6,
            "occupancy_pct": float(row[idx["sm__warps_active.avg.pct_of_peak_sustained_active"]]),
            "sm_pct": float(row[idx["sm__throughput.avg.pct_of_peak_sustained_elapsed"]]),
            "mem_pct": float(row[idx["gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"]]),
            "regs": row[idx["launch__registers_per_thread"]],
        }


def main():
    rep = sys.argv[1]
    data = list(rows(rep))
    print(f"{'kernel':60s} {'us':>8s} {'rdMB':>8s} {'wrMB':>8s} {'GB/s':>6s} {'L2MB':>8s} {'occ':>5s} {'sm%':>5s} {'mem%':>5s} regs")
    for d in data:
        gbs = (d["dram_read_MB"] + d["dram_write_MB"]) / d["time_us"] * 1e3 if d["time_us"] else 0
        print(f"{d['kernel'][:60]:60s} {d['time_us']:8.1f} {d['dram_read_MB']:8.1f} {d['dram_write_MB']:8.1f} "
              f"{gbs:6.0f} {d['l2_MB']:8.1f} {d['occupancy_pct']:5.1f} {d['sm_pct']:5.1f} {d['mem_pct']:5.1f} {d['regs']}")
    if "--csv" in sys.argv:
        with open(sys.argv[sys.argv.index("--csv") + 1], "w", newline="") as f:
            wtr = csv.DictWriter(f, fieldnames=list(data[0].keys()))
            wtr.writeheader()
            wtr.writerows(data)


if __name__ == "__main__":
    main()
