"""Per-source-line instruction / stall / shared-wavefront shares of one ncu report.

    python tools/ncu_lines.py gpurun_out/prof_stage_N9_f32.ncu-rep [top]
"""
import csv
import subprocess
import sys


def main(rep, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    cur, hdr, agg = None, None, {}
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] == "Function Name" or len(r) < 3 or r[2] != "-":
            continue
        try:
            inst = float(r[hdr.index("Instructions Executed")] or 0)
            samp = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
            wf = float(r[hdr.index("L1 Wavefronts Shared")] or 0)
            ideal = float(r[hdr.index("L1 Wavefronts Shared Ideal")] or 0)
        except (ValueError, IndexError):
            continue
        a = agg.setdefault((cur, int(r[0])), [0.0, 0.0, 0.0, 0.0, r[1][:70]])
        a[0] += inst
        a[1] += samp
        a[2] += wf
        a[3] += ideal
    ti = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    tw = sum(v[2] for v in agg.values()) or 1
    print(f"total inst {ti:.3e}  shared wavefronts {tw:.3e}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        print(f"{100*v[0]/ti:5.2f}% st {100*v[1]/ts:5.2f}% wf {100*v[2]/tw:5.2f}% (ideal {100*v[3]/tw:5.2f}) "
              f"{k[0]}:{k[1]} {v[4]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
