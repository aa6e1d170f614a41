"""Build K1 experiment variants (compile-time -D overrides) as libftk_cp_<name>.so."""
import sys
sys.path.insert(0, '.')
from paper_2011_08697_b200 import build as b
VARIANTS = {
    "base": [],
    "prof": ["FTK_K1_PROF=1"],
    "rw8": ["FTK_K1_RW=8"],
    "rw8s2": ["FTK_K1_RW=8", "FTK_K1_NSTAGE=2"],
    "rw4s4": ["FTK_K1_NSTAGE=4"],
    "rw4s6": ["FTK_K1_NSTAGE=6", "FTK_K1_MINB=1"],
}
names = sys.argv[1:] or list(VARIANTS)
for n in names:
    print(b.build_variant(n, VARIANTS[n]))
