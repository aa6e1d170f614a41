"""Build K1 experiment variants (compile-time -D overrides) as libftk_cp_<name>.so."""
import sys
sys.path.insert(0, '.')
from paper_2011_08697_b200 import build as b
VARIANTS = {
    "base": [],
    "remap": ["FTK_K1_REMAP=1"],
    "s4nb6": ["FTK_K1_NSTAGE=4", "FTK_K1_NB=6"],
    "s4nb6_remap": ["FTK_K1_NSTAGE=4", "FTK_K1_NB=6", "FTK_K1_REMAP=1"],
}
names = sys.argv[1:] or list(VARIANTS)
for n in names:
    print(b.build_variant(n, VARIANTS[n]))
