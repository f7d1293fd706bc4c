"""Summarise an ncu source page (--print-source cuda,sass CSV) by CUDA source line:
instructions executed and stall samples, top-N lines."""
import csv
import sys


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    cur_file = None
    hdr = None
    agg = []
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] == "Function Name":
            continue
        if r[2] != "-":          # sass row inside a line block
            continue
        try:
            inst = float(r[hdr.index("Instructions Executed")])
            samp = float(r[hdr.index("Warp Stall Sampling (All Samples)")])
        except (ValueError, IndexError):
            continue
        if inst or samp:
            agg.append((inst, samp, cur_file, r[0], r[1].strip()[:110]))
    tot_i = sum(a[0] for a in agg) or 1
    tot_s = sum(a[1] for a in agg) or 1
    print(f"total inst {tot_i:.3e}  samples {tot_s:.0f}")
    for a in sorted(agg, key=lambda x: -x[1])[:top]:
        print(f"{100*a[0]/tot_i:5.1f}% inst {100*a[1]/tot_s:5.1f}% stall  {a[2]}:{a[3]}  {a[4]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
