"""Build experiment variants (compile-time -D overrides) as libftk_cp_<name>.so, selected at run time
with FTK_LIB=<path> (tools/gpu_var.sh, tools/var_time.sh).  usage: python tools/variants.py name..."""
import sys
sys.path.insert(0, '.')
from paper_2011_08697_b200 import build as b
VARIANTS = {
    "base": [],
    "checks": ["FTK_CHECKS=1"],             # device assertions (tools/checks_run.sh)
    "prof": ["FTK_K1_PROF=1"],              # K1 cycle accounting in counters[CNT_PROF..]
    "xminb3": ["FTK_X_MINB=3"],             # k_exact2d occupancy
    "rw4": ["FTK_K1_RW=4"],                 # k_scan2d rows per warp
    "tch16": ["FTK_K1_TCHUNK=16"],          # k_scan2d timesteps per work item (halved for small grids)
    "gsr0": ["FTK_GATHER_SR=0"],            # byte-pick gather instead of sign-replicating PRMT
    "s3r0": ["FTK_S3_REGION=0"],            # k_scan3d without the region test
    "s3cnt": ["FTK_S3_COUNT=1"],            # region-test statistics in counters[CNT_PROF..]
    "s3noc": ["FTK_S3_NOCODES=1"],          # k_scan3d timing floor without per-vertex codes (results invalid)
    "s3sp2": ["FTK_S3_SPLIT=2"],            # two scan warps per z-slice
    "s3tp1": ["FTK_S3_TP=1"],               # one squares task per slice
    "s3tp4": ["FTK_S3_TP=4"],
    "x3m4": ["FTK_X3_MINB=4"],              # k_exact3d occupancy
    "jump2": ["FTK_LABEL_JUMP=2"],          # pointer jumping before k_label
    "hrun128": ["FTK_HRUN=128"],            # pass-2 hash: slots probed per block before a jump
    "hrun512": ["FTK_HRUN=512"],
    "ufkey": ["FTK_UF_PRIO=0"],              # union-find linked by face id (round-1 design)
}
names = sys.argv[1:] or list(VARIANTS)
for n in names:
    print(b.build_variant(n, VARIANTS[n]))
