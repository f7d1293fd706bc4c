"""Per-launch DRAM bytes and device time of the bbdg kernels in an ncu launch list taken on the
HBM-filling bench (--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum),
merged into profiles/traffic.json["fill"][dtype][N] for the stage kernel of each order (the bench's
roofline.traffic) and printed per kernel family (volume / surface / stage / update)."""
import csv
import json
import re
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OPS = {"0": "volume", "1": "surface", "2": "rhs", "3": "stage"}


def to_bytes(v, unit):
    return float(v.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main(path, box_k_json=None):
    rows = list(csv.DictReader([ln for ln in open(path) if not ln.startswith("==")]))
    per = defaultdict(lambda: defaultdict(dict))
    for r in rows:
        per[r["ID"]][r["Metric Name"]] = (r["Metric Value"], r["Metric Unit"])
        per[r["ID"]]["name"] = r["Kernel Name"]
    fam = defaultdict(list)
    for lid, m in per.items():
        name = m["name"]
        mo = re.match(r"void (?:bbdg::)?(opt_kernel|ept_kernel)<(float|double), (\d), (\d)", name)
        mu = re.match(r"void (?:bbdg::)?lsrk_update_vec_kernel<(float|double)", name)
        if mo:
            key = (mo.group(2), int(mo.group(3)), OPS[mo.group(4)])
        elif mu:
            key = (mu.group(1), 0, "update")
        else:
            continue
        rd = to_bytes(*m["dram__bytes_read.sum"]) if "dram__bytes_read.sum" in m else 0.0
        wr = to_bytes(*m["dram__bytes_write.sum"]) if "dram__bytes_write.sum" in m else 0.0
        t = float(m["gpu__time_duration.sum"][0].replace(",", ""))
        t *= {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(m["gpu__time_duration.sum"][1], 1.0)
        fam[key].append((rd + wr, t))
    out = {}
    for (dt, N, op), v in sorted(fam.items()):
        b = sum(x[0] for x in v) / len(v)
        t = sum(x[1] for x in v) / len(v)
        print(f"{dt:6s} N={N} {op:8s} launches {len(v):3d}  dram {b / 1e9:9.3f} GB/launch  {t / 1e3:8.3f} ms  "
              f"{b / (t * 1e-6) / 1e9:8.1f} GB/s (cold, serialised)")
        if op == "stage":
            out.setdefault("f32" if dt == "float" else "f64", {})[str(N)] = {"dram_bytes": b, "ncu_ms": t / 1e3}
    if box_k_json:   # K of each order's mesh, from the bench line that ran under ncu
        d = json.loads(Path(box_k_json).read_text().strip().splitlines()[-1])
        for dn, r in d["per_dtype"].items():
            for N, row in r["per_order"].items():
                if dn in out and N in out[dn]:
                    out[dn][N]["K"] = row["K"]
    tp = ROOT / "profiles" / "traffic.json"
    data = json.loads(tp.read_text()) if tp.exists() else {}
    data.setdefault("fill", {})
    for dn, v in out.items():
        data["fill"].setdefault(dn, {}).update(v)
    tp.write_text(json.dumps(data, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
