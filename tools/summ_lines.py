"""Summarise bench JSON lines (one per file): step, sweep, e2e, roofline."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        r = d["roofline"]
        t = r["terms"]
        e2e = d["e2e"].get("ms_per_step", d["e2e"].get("value"))
        print(f"{f:40s} step {d['ms_per_step']:.3f} sweep {t['t_sweep_ms']:.3f} e2e {e2e:.3f} "
              f"{r['bound']} {r['frac']:.3f} lines/red {t.get('mean_lines_per_red_instr', 0):.2f}")
    except Exception as e:  # noqa: BLE001
        print(f, "ERR", e)
