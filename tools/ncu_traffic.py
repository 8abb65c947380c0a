"""Per-kernel-kind DRAM traffic from an ncu report of one build.

    python tools/ncu_traffic.py gpurun_out/ncu_X.ncu-rep <workload> [--out profiles/ncu_traffic.json] [--csv summary.csv]

Maps each launch to the kernel kinds bench.py reports (dmst.cu KernelKind)
and records, per kind, launches, device time and dram__bytes_read +
dram__bytes_write per launch (bench.py's roofline.traffic).  ncu times are
cold-cache and serialised: use the shares, not the absolutes.
"""
import csv
import json
import subprocess
import sys

METS = "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
TS = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
BS = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def kind(name: str) -> str:
    rules = [
        ("k_local_final", "sort1_local"),
        ("k_key_reduce", "sort1_hist"), ("k_upsweep", "upsweep_scan"), ("k_row_scan", "upsweep_scan"), ("k_row_total_scan", "upsweep_scan"),
        ("Sort1Loader", "sort1_pass_first"), ("Sort1Emitter", "sort1_pass_final"),
        ("Sort1FirstLoader", "sort1_pass_first"), ("Sort1FinalEmitter", "sort1_pass_final"),
        ("k_downsweep<unsigned long, 0,", "sort2_pass"), ("k_downsweep<unsigned long", "sort1_pass_mid"),
        ("k_downsweep<unsigned int, 3,", "sort1_pass_mid"),
        ("k_downsweep<unsigned int", "sort2_pass"),
        ("k_fine_hist", "mi_hist"), ("k_fine_scan", "mi_hist"),
        ("k_split<0, EdgeRecSrc", "mi_split_a"), ("k_split<1, AosRecSrc<3>", "mi_split_b"),
        ("LinkSortedSrc", "link_split"), ("k_split<1, AosRecSrc<2>", "link_split"), ("k_link_cursors", "link_split"),
        ("k_link_apply", "link_apply"), ("k_link(", "link_apply"),
        # sliced maxIncident (views 0/1): k_mi_atomic + k_v1 are bench.py's mi_apply; ncu cannot
        # tell a sliced view's k_v1 from a direct view's, so all k_v1 launches stay "v1" here
        ("k_mi_apply_smem", "mi_apply"), ("k_mi_atomic", "mi_apply"), ("k_slice_scan", "mi_hist"),
        ("k_link_scatter", "link_apply"), ("k_ls_", "leafscan"), ("k_v1", "v1"), ("k_leafscan", "leafscan"), ("k_v2", "v2"),
        ("k_jump", "jump"), ("k_select_edges", "select_edges"), ("k_walk", "walk"), ("k_tail", "tail"),
        ("k_key_sample", "sort1_hist"),
        # outside the timed build: bench.py's validation leg, statistics
        ("k_validate_scan", "validate"), ("k_cc_", "validate"), ("k_adjacent_equal", "validate"),
        ("k_depth_", "stats"), ("k_count_heads", "stats"),
    ]
    for pat, k in rules:
        if pat in name:
            return k
    return "other"


def main():
    rep, workload = sys.argv[1], sys.argv[2]
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
    if rep.endswith(".csv"):  # a saved `ncu -i X --page raw --csv --metrics METS` export
        raw = open(rep).read()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", METS],
                             capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    h, units = r[0], r[1]
    ix = {k: i for i, k in enumerate(h)}
    agg = {}
    for row in r[2:]:
        k = kind(row[ix["Kernel Name"]])
        t = float(row[ix["gpu__time_duration.sum"]].replace(",", "")) * TS[units[ix["gpu__time_duration.sum"]]]
        b = sum(float(row[ix[m]].replace(",", "")) * BS[units[ix[m]]]
                for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        a = agg.setdefault(k, {"launches": 0, "time_us": 0.0, "dram_bytes": 0.0})
        a["launches"] += 1
        a["time_us"] += t
        a["dram_bytes"] += b
    tot = sum(a["time_us"] for a in agg.values())
    summary = {}
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["time_us"]):
        summary[k] = {"launches": a["launches"], "time_us": round(a["time_us"], 1),
                      "share": round(a["time_us"] / tot, 4),
                      "dram_bytes_per_launch": a["dram_bytes"] / a["launches"],
                      "dram_GBs": a["dram_bytes"] / (a["time_us"] * 1e-6) / 1e9 if a["time_us"] else 0.0}
        print(f"{k:18s} {a['launches']:4d} launches {a['time_us']:9.1f} us ({a['time_us'] / tot * 100:5.1f}%)  "
              f"DRAM {a['dram_bytes'] / 1e9:7.2f} GB  {summary[k]['dram_GBs']:7.0f} GB/s")
    if out:
        try:
            cur = json.load(open(out))
        except Exception:
            cur = {}
        cur[workload] = {k: v["dram_bytes_per_launch"] for k, v in summary.items()}
        cur.setdefault("_detail", {})[workload] = summary
        json.dump(cur, open(out, "w"), indent=1)
    if "--csv" in sys.argv:
        with open(sys.argv[sys.argv.index("--csv") + 1], "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["kind", "launches", "time_us", "share", "dram_bytes_per_launch", "dram_GBs"])
            for k, v in summary.items():
                w.writerow([k, v["launches"], v["time_us"], v["share"], int(v["dram_bytes_per_launch"]),
                            round(v["dram_GBs"], 1)])


if __name__ == "__main__":
    main()
