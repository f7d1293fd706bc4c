"""Aggregate an ncu source page (--print-source cuda,sass --csv) per CUDA source line:
python tools/src_lines.py report.csv [top]  -> top lines by shared wavefronts / stall samples."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
agg = collections.defaultdict(lambda: collections.Counter())
text = {}
fname = None
hdr = None
cur = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "Function Name":
        continue
    if r[0]:   # a source line row
        cur = (fname, int(r[0]))
        text[cur] = r[1][:70]
        continue
    if cur is None:
        continue
    d = dict(zip(hdr[2:], r[2:]))
    for k in ("Warp Stall Sampling (All Samples)", "L1 Wavefronts Shared", "L1 Wavefronts Shared Excessive",
              "Instructions Executed"):
        try:
            agg[cur][k] += float(d.get(k) or 0)
        except ValueError:
            pass
tot = collections.Counter()
for v in agg.values():
    tot.update(v)
print({k: f"{v:.3g}" for k, v in tot.items()})
for key in ("L1 Wavefronts Shared", "Warp Stall Sampling (All Samples)"):
    print(f"\n== top by {key}")
    for ln, v in sorted(agg.items(), key=lambda kv: -kv[1][key])[:top]:
        print(f"{100 * v[key] / max(tot[key], 1):5.1f}%  wf {v['L1 Wavefronts Shared']:.3g} exc "
              f"{v['L1 Wavefronts Shared Excessive']:.3g} st {v['Warp Stall Sampling (All Samples)']:.0f} "
              f"inst {v['Instructions Executed']:.3g}  {ln[0]}:{ln[1]}  {text.get(ln, '')}")
