"""Summarise bench JSON lines: python tools/bsum.py file.json ..."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable", e)
        continue
    r = d.get("roofline") or {}
    pk = r.get("per_kernel", {})
    ks = " ".join(f"{k}={v['ms']*1e3:.0f}us/{v['frac']:.3f}" for k, v in pk.items())
    print(f"{f}: {d['config'].get('name')} {d['value']/1e6:.2f} M/s {d['ms_per_step']:.4f} ms "
          f"e2e {d.get('e2e', {}).get('value', 0)/1e6:.2f} | {ks}")
