"""Stall samples and executed instructions of an ncu --set full capture,
aggregated by CUDA source line (needs -lineinfo and --import-source on):
python tools/ncu_by_line.py gpurun_out/r02_sweep_c5.ncu-rep [top]"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(r for r in rows if r and r[0] == "Line No")
    i_line, i_ss, i_ie = 0, hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    agg = {}
    cur = None
    src = {}
    fname = ""
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
            continue
        if r[0] in ("Function Name", "Line No"):
            continue
        if r[0].strip():  # a CUDA source line row
            cur = (fname, int(r[0]))
            src[cur] = r[1]
        elif cur is not None and len(r) > i_ss and r[i_ss] not in ("", "-"):
            s, e = agg.get(cur, (0, 0))
            agg[cur] = (s + int(r[i_ss]), e + int(r[i_ie] if r[i_ie] not in ("", "-") else 0))
    tot_s = sum(v[0] for v in agg.values()) or 1
    tot_e = sum(v[1] for v in agg.values()) or 1
    print(f"total stall samples {tot_s}, warp instructions {tot_e}")
    for ln, (s, e) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{ln[0][:12]}:{ln[1]:<5d} {100 * s / tot_s:5.1f}% samples {100 * e / tot_e:5.1f}% instr  {src.get(ln, '').strip()[:90]}")


if __name__ == "__main__":
    main()
