"""Split an ncu source page (cuda,sass CSV) into kernel phases by source-line ranges of
bbdg_tile.cuh, using the phase marker comments in the kernel."""
import csv
import re
import sys

MARK = {"S1:": "S1 flux", "S2:": "S2 L0", "S3 (optimal": "S3 cascade", "dense lift input": "S2 dense-in",
        "volume V1": "V1", "V2 + surface gather": "V2+EP", "staged views": "stage/wait", "producer:": "producer"}


def main(path, src):
    lines = open(src).read().splitlines()
    kern = next(i for i, l in enumerate(lines) if "the kernel" in l) + 1
    marks = []
    for i, l in enumerate(lines):
        for k, v in MARK.items():
            if k in l and i > kern:
                marks.append((i + 1, v))
    marks.sort()
    rows = list(csv.reader(open(path)))
    cur = None
    hdr = None
    agg = {}
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] == "Function Name" or r[2] != "-":
            continue
        try:
            inst = float(r[hdr.index("Instructions Executed")])
            samp = float(r[hdr.index("Warp Stall Sampling (All Samples)")])
        except (ValueError, IndexError):
            continue
        ln = int(r[0])
        ph = "other/helpers"
        if cur == "bbdg_tile.cuh" and ln > kern:
            for m, v in marks:
                if ln >= m:
                    ph = v
        elif cur == "bbdg_tile.cuh":
            ph = "helpers/tables"
        a = agg.setdefault(ph, [0.0, 0.0])
        a[0] += inst
        a[1] += samp
    ti = sum(v[0] for v in agg.values())
    ts = sum(v[1] for v in agg.values())
    for k, v in sorted(agg.items(), key=lambda x: -x[1][0]):
        print(f"{k:16s} inst {100*v[0]/ti:5.1f}%  stall {100*v[1]/ts:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
