"""Build K1 experiment variants (compile-time -D overrides) as libftk_cp_<name>.so."""
import sys
sys.path.insert(0, '.')
from paper_2011_08697_b200 import build as b
VARIANTS = {
    "base": [],
    "static": ["FTK_K1_DYN=0"],
    "new4": ["FTK_K1_NEW=4"],
    "new2": ["FTK_K1_NEW=2"],
    "prof": ["FTK_K1_PROF=1"],
    "nocopy": ["FTK_K1_PROF=1", "FTK_K1_DIAG_NOCOPY=1"],
    "noexact": ["FTK_K1_PROF=1", "FTK_K1_DIAG_NOEXACT=1"],
    "nocopy_noexact": ["FTK_K1_PROF=1", "FTK_K1_DIAG_NOCOPY=1", "FTK_K1_DIAG_NOEXACT=1"],
    "prof_new4": ["FTK_K1_PROF=1", "FTK_K1_NEW=4"],
}
names = sys.argv[1:] or list(VARIANTS)
for n in names:
    print(b.build_variant(n, VARIANTS[n]))
