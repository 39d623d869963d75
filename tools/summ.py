"""Summarise bench JSON lines: python tools/summ.py gpurun_out/TAG_c*.json"""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as exc:  # noqa: BLE001
        print(f, "unreadable", exc)
        continue
    r = d["roofline"]
    t = r["terms"]
    print(f"{d['config']['workload'][:8]} step {d['ms_per_step']:.3f} ms  sweep {r['sweep_ms']:.3f}  "
          f"e2e {d['e2e']['ms_per_step']:.3f}  bound {r['bound']} frac {r['frac']:.3f}  "
          f"fp64 {t['t_fp64_ms']:.3f}  red {t.get('t_red_ms', float('nan')):.3f}  "
          f"reds {t['reds']:.3g} lines/instr {t.get('mean_lines_per_red_instr', float('nan')):.2f} "
          f"records {t.get('red_records', 0):.3g} shape-priced {t.get('t_red_shape_priced_ms', float('nan')):.3f}")
