"""Build f32 tuning variants of the library (different tile shapes / group counts)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1512_06025_b200.build import build_variant  # noqa: E402

F64 = {"vH", "vI"}
VARIANTS = {
    "vJ": ["-DBBDG_OPT_NG_TMEM=6"],
    "vK": ["-DBBDG_OPT_NG_TMEM=6", "-DBBDG_OPT_TMEM_MIN_N=2"],
    "vH": ["-DBBDG_OPT_KE8=0,16,12,6,4,3,2,2,1,1"],
    "vI": ["-DBBDG_OPT_KE8=0,32,24,12,6,4,3,2,2,1"],
    "vB": ["-DBBDG_OPT_KE4=0,16,12,6,4,2,2,1,1,1", "-DBBDG_OPT_NG4=0,8,8,8,6,6,6,4,4,4"],
    "vC": ["-DBBDG_OPT_KE4=0,32,24,12,6,4,3,2,2,1", "-DBBDG_OPT_NG4=0,4,4,4,4,4,4,4,3,4"],
    "vD": ["-DBBDG_OPT_KE4=0,8,6,4,2,2,1,1,1,1", "-DBBDG_OPT_NG4=0,8,8,8,8,8,8,6,6,5"],
    "vE": ["-DBBDG_OPT_KE4=0,32,24,12,6,6,4,3,2,2", "-DBBDG_OPT_NG4=0,4,4,4,4,4,4,3,3,3"],
    "vS": ["-DBBDG_OPT_NG_SURF=6"],
    "vF": ["-DBBDG_OPT_KE4=0,32,24,12,6,4,3,2,2,1", "-DBBDG_OPT_NG4=0,5,5,5,5,5,5,5,3,5"],
    "vG": ["-DBBDG_OPT_KE4=0,32,24,12,6,4,3,2,2,1", "-DBBDG_OPT_NG4=0,6,6,6,6,6,6,6,4,6"],
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(VARIANTS)
    for n in names:
        d = Path("variants").resolve() / n
        d.mkdir(parents=True, exist_ok=True)
        hdr = d / "tune.h"
        hdr.write_text("".join(f"#define {x[2:].split('=')[0]} {x.split('=', 1)[1]}\n" for x in VARIANTS[n]))
        print(n, build_variant(d, ["--pre-include", str(hdr)], dtypes=("f64",) if n in F64 else ("f32",)))
