"""Copy a GPU evidence run (tools/gpu/run_evidence.sh, TAG) into profiles/
and regenerate DESIGN.md §7's table between the RESULTS markers:
    python tools/refresh_results.py r02c"""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def last_json(path):
    return json.loads(open(path).read().strip().splitlines()[-1])


def main(tag):
    shutil.copy(os.path.join(OUT, f"{tag}_bench.json"), os.path.join(PROF, "r02_bench.json"))
    shutil.copy(os.path.join(OUT, f"{tag}_bench_ref.json"), os.path.join(PROF, "r02_bench_reference.json"))
    shutil.copy(os.path.join(OUT, f"{tag}_launches.csv"), os.path.join(PROF, "r02_launches.csv"))
    shutil.copy(os.path.join(OUT, f"{tag}_gputests.log"), os.path.join(PROF, "r02_gputests.log"))
    rows = list(csv.reader(open(os.path.join(PROF, "r02_launches.csv"))))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[start + 1:]:
        agg[r[ki].split("(")[0]][0] += 1
        agg[r[ki].split("(")[0]][1] += float(r[vi].replace(",", ""))
    tot = sum(a[1] for a in agg.values())
    out = ["ncu --metrics gpu__time_duration.sum --clock-control none of:",
           "  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-per-config --no-red-trace",
           "(config 5 headline; cold-cache, serialised replay: absolute times are not bench times, the SHARE is.",
           " sweep_kernel<2,1,...> is the untimed DIAG=1 counting launch; the timed step is the staged",
           " sweep_kernel<2,0,1,64,64,1> (phase 1) + sweep_units_kernel (phase 2) + zcap_kernel (cap refresh)",
           " sequence of the capped sub-strips, fill / decode / areal / profiles)",
           f"total kernel time {tot / 1e6:.2f} ms over {sum(a[0] for a in agg.values())} launches", ""]
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"{a[1] / 1e6:10.3f} ms {100 * a[1] / tot:6.2f} %  {a[0]:6d} launches  {k[:110]}")
    open(os.path.join(PROF, "r02_launches_summary.txt"), "w").write("\n".join(out) + "\n")
    summ = [f"round-2 ncu --set full captures (--clock-control none), tools/ncu_summary.py; commands: "
            f"tools/gpu/run_evidence.sh (TAG={tag})"]
    for f in ("units_c5", "p1_c5", "sweep_c3", "sweep_c4", "sweep_c2"):
        rep = os.path.join(OUT, f"{tag}_{f}.ncu-rep")
        summ.append(f"=== {tag}_{f}")
        summ.append(subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep],
                                   capture_output=True, text=True).stdout)
    for f, what in (("units_c5", "config 5 phase-2 units kernel"), ("p1_c5", "config 5 staged phase-1 kernel")):
        summ.append(f"=== hot source lines, {what}")
        summ.append(subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_by_line.py"),
                                    os.path.join(OUT, f"{tag}_{f}.ncu-rep"), "15"], capture_output=True, text=True).stdout)
    open(os.path.join(PROF, "r02_ncu_summary.txt"), "w").write("\n".join(summ))

    d = last_json(os.path.join(PROF, "r02_bench.json"))
    ref = last_json(os.path.join(PROF, "r02_bench_reference.json"))
    upd = {"config1": 5.76e7, "config2": 1.58e9, "config3": 4.95e10, "config4": 4.12e9}
    tab = ["| workload | updates / step | device step | sweep | value (updates/s) | e2e step | e2e (updates/s) | "
           "roofline bound, frac | CPU reference (16 threads) |", "|---|---|---|---|---|---|---|---|---|"]

    def row(name, v, u):
        rf, cb = v["roofline"], v.get("cpu_baseline") or {}
        return (f"| {name} | {u:.3g} | {v['ms_per_step']:.3f} ms | {rf['sweep_ms']:.3f} ms | {v['value']:.3g} | "
                f"{v['e2e']['ms_per_step']:.3f} ms | {v['e2e']['value']:.3g} | {rf['bound']} {rf['frac']:.2f} | "
                f"{cb.get('value', float('nan')):.3g} |")

    tab.append(row("**config 5** (headline: ball R2, tilt, noise, 16 passes, 4096²)", d,
                   d["config"]["edge_point_updates_per_surface"]))
    for k, v in d["per_config"].items():
        tab.append(row(k, v, upd[k]))
    tab.append("")
    tab.append(f"Reference arm (`bench.py --impl reference`: the reference algorithm restated in oracle/, "
               f"{ref['cpu_baseline']['cores']} host threads, config 5 bounded sample): {ref['value']:.3g} updates/s; "
               f"the headline e2e through the public API is {d['e2e']['value'] / ref['value']:.0f}x that, the "
               f"device value {d['value'] / ref['value']:.0f}x. Clocks {d['clocks']['sm_mhz']:.0f} MHz, throttle "
               f"reasons {d['clocks']['reasons'] or 'none'}.")
    s = open(os.path.join(ROOT, "DESIGN.md")).read()
    a = s.index("<!-- RESULTS -->") + len("<!-- RESULTS -->")
    b = s.index("<!-- /RESULTS -->")
    s = s[:a] + "\n" + "\n".join(tab) + "\n" + s[b:]
    open(os.path.join(ROOT, "DESIGN.md"), "w").write(s)
    print("\n".join(tab))


if __name__ == "__main__":
    main(sys.argv[1])
