"""Build f32 tuning variants of the library (different tile shapes / group counts)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1512_06025_b200.build import build_variant  # noqa: E402

F64 = {"e8", "f8", "ept64", "loc64", "nonb64"}
BOTH = {"eptold"}
VARIANTS = {
    "k2": ["-DBBDG_OPT_KE4=0,32,16,12,6,4,3,2,2,1"],   # fp32 N=2: KE 16
    "k3": ["-DBBDG_OPT_KE4=0,32,24,8,6,4,3,2,2,1"],    # fp32 N=3: KE 8
    "keup": ["-DBBDG_OPT_KE4=0,32,16,12,6,5,4,3,3,2"],   # fp32 N >= 5: one more element per tile
    "kedn": ["-DBBDG_OPT_KE4=0,32,16,12,6,3,2,2,1,1"],   # fp32 N >= 5: one fewer
    "ng4": ["-DBBDG_OPT_NG_TMEM=4"],                     # TMEM-mode groups per CTA
    "ng6": ["-DBBDG_OPT_NG_TMEM=6"],
    "a4": ["-DBBDG_OPT_KE4=0,32,16,12,4,4,3,3,2,1"],          # fp32 N=4: KE 4
    "b4": ["-DBBDG_OPT_KE4=0,32,16,12,8,4,3,3,2,1"],          # fp32 N=4: KE 8
    "c4": ["-DBBDG_OPT_NGT4=0,5,5,5,4,4,4,4,5,5"],            # fp32 N=4,5: 4 groups
    "d4": ["-DBBDG_OPT_NGT4=0,5,5,5,6,6,4,4,4,4"],            # fp32 N=4,5: 6 groups, N=8,9: 4
    "e8": ["-DBBDG_OPT_KE8=0,16,12,6,5,3,3,3,2,2"],           # fp64 N >= 4: one more element per tile
    "f8": ["-DBBDG_OPT_NGT8=0,4,4,5,5,5,5,5,5,5"],            # fp64 TMEM-mode groups 5 at N >= 4
    "ept64": ["-DBBDG_EPT_MAX_N64=3"],                         # fp64 N=3 on the register kernel
    "ept4": ["-DBBDG_EPT_MAX_N=4"],                            # fp32 N=4 on the register kernel
    "nonb": ["-DBBDG_EXP_NO_NB=1"],
    "nonb64": ["-DBBDG_EXP_NO_NB=1"],
    "eptold": ["-DBBDG_EPT_LOCNB=0"],
    "kc8": ["-DBBDG_TC_KC=8"],                                 # tcgen05 nodal: 8-wide K chunks (more stages)
    "kc32": ["-DBBDG_TC_KC=32"],                               # tcgen05 nodal: 32-wide K chunks
    "shf2": ["-DBBDG_OPT_SHF4=0,1,1,1,2,2,2,2,2,2"],          # cascade levels read by shuffles up to 2 parent slots
    "shf0": ["-DBBDG_OPT_SHF4=0,0,0,0,0,0,0,0,0,0"],          # no shuffle levels                          # EPT without the in-tile neighbour copies
    "loc64": ["-DBBDG_OPT_LOCNB8=0,0,0,1,1,1,1,1,1,1"],        # fp64: in-tile neighbour traces at N >= 3                              # experiment: no neighbour gather (wrong results)
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(VARIANTS)
    for n in names:
        d = Path("variants").resolve() / n
        d.mkdir(parents=True, exist_ok=True)
        hdr = d / "tune.h"
        hdr.write_text("".join(f"#define {x[2:].split('=')[0]} {x.split('=', 1)[1]}\n" for x in VARIANTS[n]))
        print(n, build_variant(d, ["--pre-include", str(hdr)], dtypes=("f32", "f64") if n in BOTH else (("f64",) if n in F64 else ("f32",))))
