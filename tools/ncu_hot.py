"""Top SASS instructions by warp-stall samples from an ncu --page source --csv dump."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = None
data = []
for r in rows:
    if len(r) > 3 and r[0] == "Address":
        hdr = {k: i for i, k in enumerate(r)}
        continue
    if hdr and len(r) == len(hdr):
        data.append(r)
S = hdr["Warp Stall Sampling (All Samples)"]
tot = sum(int(r[S] or 0) for r in data)
wf = hdr.get("L1 Wavefronts Shared")
wfi = hdr.get("L1 Wavefronts Shared Ideal")
print(f"total samples {tot}")
for r in sorted(data, key=lambda r: -int(r[S] or 0))[:top]:
    extra = f" smem wf {r[wf]}/{r[wfi]}" if wf is not None and r[wf] not in ("0", "") else ""
    print(f"{int(r[S]) / tot * 100:5.1f}%  {r[hdr['Address']][-5:]}  {r[hdr['Source']].strip()[:70]}{extra}")
