"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): total device
time per kernel family and each family's share of all launches."""
import csv
import re
import sys
from collections import defaultdict


def family(name):
    m = re.match(r"void (?:bbdg::)?(\w+)<([^>]*)>", name)
    if m:
        return f"bbdg::{m.group(1)}<{m.group(2)}>"
    return "torch/other: " + name.split("(")[0][:60]


def main(path):
    lines = [ln for ln in open(path) if not ln.startswith("==")]
    rows = list(csv.DictReader(lines))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        if r["Metric Unit"] == "us":
            v *= 1e3
        elif r["Metric Unit"] == "ms":
            v *= 1e6
        f = family(r["Kernel Name"])
        tot[f] += v
        cnt[f] += 1
    all_t = sum(tot.values())
    ours = sum(v for k, v in tot.items() if k.startswith("bbdg::"))
    print(f"launches: {sum(cnt.values())}, device time {all_t/1e6:.3f} ms, bbdg kernels {100*ours/all_t:.1f}%")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{100*v/all_t:6.2f}%  {v/1e6:9.4f} ms  x{cnt[k]:4d}  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
