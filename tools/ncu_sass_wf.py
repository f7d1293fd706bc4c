"""Shared-memory wavefronts per SASS instruction (deduplicated by address) with the source
line ncu attributes it to.   python tools/ncu_sass_wf.py rep.ncu-rep [top] [elements]"""
import csv
import subprocess
import sys


def main(rep, top=30, K=105456):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, cur, seen, res = None, None, set(), []
    for r in rows:
        if not r:
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] in ("File Path", "Function Name"):
            continue
        if len(r) > 3 and r[2].startswith("0x"):
            if r[2] in seen:
                continue
            seen.add(r[2])
            try:
                wf = float(r[hdr.index("L1 Wavefronts Shared")] or 0)
                ideal = float(r[hdr.index("L1 Wavefronts Shared Ideal")] or 0)
                ex = float(r[hdr.index("Instructions Executed")] or 0)
            except (ValueError, IndexError):
                continue
            if wf > 0:
                res.append((wf, ideal, ex, cur, r[3].strip()[:48]))
        else:
            cur = f"{r[0]}: {r[1].strip()[:60]}"
    tot = sum(x[0] for x in res)
    print(f"total shared wavefronts {tot:.4e} = {tot / K:.0f} per element; ideal {sum(x[1] for x in res) / K:.0f}")
    agg = {}
    for wf, ideal, ex, line, s in res:
        a = agg.setdefault(line, [0.0, 0.0, 0])
        a[0] += wf
        a[1] += ideal
        a[2] += 1
    for line, (wf, ideal, n) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        print(f"{wf / K:7.1f} wf/elem (ideal {ideal / K:6.1f}, {n:3d} instr)  {line}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
