"""Summarise bench lines of an A/B directory: value, e2e, per-axis ms, frac."""
import glob, json, os, sys
for f in sorted(glob.glob(os.path.join(sys.argv[1], "bench_*.json"))):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(os.path.basename(f), "ERR", e); continue
    r = d.get("roofline", {})
    print(f"{os.path.basename(f):40s} {d['value']:7.2f}  e2e {d['e2e']['value']:6.2f}  axes "
          + "/".join(f"{x:.3f}" for x in r.get("per_axis_ms_in_step", []))
          + f"  frac {r.get('frac', 0):.3f}")
