"""Print a one-screen summary of a bench.py JSON line (ms/step, per-kernel ms)."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable:", e)
        continue
    c = d.get("config", {})
    print(f"{f}: {d['ms_per_step']:.3f} ms/step, {d['value']:.3e} {d['unit']}, frac "
          f"{d.get('pipeline_roofline', {}).get('frac', 0):.3f}, e2e {d.get('e2e', {}).get('value', 0):.3e} "
          f"(serial {d.get('e2e', {}).get('serial', {}).get('value', 0):.3e}), "
          f"paths {c.get('paths')} L {c.get('levels')} parity {d.get('parity')}")
    print("   ", {k: round(v, 3) for k, v in d.get("kernel_ms_per_step", {}).items()})
