"""Summarise an ncu --set full report of the sweep kernel (run here, no GPU):
python tools/ncu_summary.py gpurun_out/sweep_r01b.ncu-rep [--sass N]"""
import csv
import io
import subprocess
import sys


def ncu(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep = sys.argv[1]
    rows = ncu(rep, "--page", "raw")
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    keys = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__occupancy_limit_registers", "smsp__inst_executed.sum",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
            "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "lts__t_requests_srcunit_l1_op_red.sum",
            "lts__t_requests_srcunit_l1_op_atom.sum", "smsp__thread_inst_executed_per_inst_executed.ratio"]
    for k in keys:
        if k in d:
            print(f"{k:70s} {d[k]} {u.get(k, '')}")
    st = sorted(((k, float(v)) for k, v in d.items()
                 if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
                 and v not in ("", "n/a")), key=lambda kv: -kv[1])
    print("stall reasons (warps per issue):")
    for k, v in st[:10]:
        print(f"   {k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]:28s} {v:.3f}")
    pipes = sorted(((k, v) for k, v in d.items() if k.startswith("sm__inst_executed_pipe_") and k.endswith(".avg.pct_of_peak_sustained_active")), key=lambda kv: -float(kv[1] or 0))
    print("pipe utilisation (% of peak, active):")
    for k, v in pipes[:8]:
        print(f"   {k[len('sm__inst_executed_pipe_'):-len('.avg.pct_of_peak_sustained_active')]:28s} {v}")
    if "--sass" in sys.argv:
        n = int(sys.argv[sys.argv.index("--sass") + 1])
        src = ncu(rep, "--page", "source", "--print-source", "sass")
        h = src[1]
        ia, isrc, iss = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
        data = src[2:]
        tot = sum(int(r[iss] or 0) for r in data)
        top = sorted(data, key=lambda r: -int(r[iss] or 0))[:n]
        print(f"top {n} SASS lines by stall samples (total {tot}):")
        for r in top:
            print(f"   {int(r[iss]):7d} {int(r[ia] or 0):11d}  {r[isrc].strip()[:80]}")


if __name__ == "__main__":
    main()
