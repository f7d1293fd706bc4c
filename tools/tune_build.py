"""Build f32 tuning variants of the library (different tile shapes / group counts)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1512_06025_b200.build import build_variant  # noqa: E402

F64 = {"m3d", "m4d"}
VARIANTS = {
    "m3d": ["-DBBDG_OPT_TMEM64_MIN_N=3", "-DBBDG_OPT_NGT8=0,4,4,5,5,5,4,4,4,4"],   # fp64 N=3, 4: 5 TMEM groups
    "m4d": ["-DBBDG_OPT_NGT8=0,4,4,4,5,5,4,4,4,4"],                              # fp64 N=4: 5 groups
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(VARIANTS)
    for n in names:
        d = Path("variants").resolve() / n
        d.mkdir(parents=True, exist_ok=True)
        hdr = d / "tune.h"
        hdr.write_text("".join(f"#define {x[2:].split('=')[0]} {x.split('=', 1)[1]}\n" for x in VARIANTS[n]))
        print(n, build_variant(d, ["--pre-include", str(hdr)], dtypes=("f64",) if n in F64 else ("f32",)))
