"""Opcode mix (share of executed warp instructions) of one ncu report's SASS page."""
import csv
import subprocess
import sys
from collections import Counter


def main(rep, K=105456):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    ii = hdr.index("Instructions Executed")
    c = Counter()
    for r in rows[2:]:
        if len(r) <= ii:
            continue
        s = r[1].strip()
        op = (s.split()[1] if s.startswith("@") else s.split()[0]).split(".")[0]
        c[op] += float(r[ii] or 0)
    tot = sum(c.values())
    print(f"total {tot:.4e} warp-inst, {tot / K:.0f} per element")
    print("  ".join(f"{op} {100 * n / tot:.1f}" for op, n in c.most_common(28)))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 105456)
