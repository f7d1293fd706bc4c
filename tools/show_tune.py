import glob
import json
for f in sorted(glob.glob("gpurun_out/tune_*.json")):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "ERR", open(f.replace(".json", ".err")).read()[-300:])
        continue
    print(f"{f:32s} {d['value']:7.2f}", " ".join(f"{r['gdofs_stage']:6.1f}" for r in d["per_order"].values()))
