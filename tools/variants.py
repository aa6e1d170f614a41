"""Build K1 experiment variants (compile-time -D overrides) as libftk_cp_<name>.so."""
import sys
sys.path.insert(0, '.')
from paper_2011_08697_b200 import build as b
VARIANTS = {
    "base": [],
    "prof": ["FTK_K1_PROF=1"],
    "mixhash": ["FTK_LOCAL_HASH=0"],
    "xminb2": ["FTK_X_MINB=2"],
    "xminb4": ["FTK_X_MINB=4"],
    "s2m3": ["FTK_K1_NSTAGE=2", "FTK_K1_MINB=3"],
    "rw4": ["FTK_K1_RW=4"],
    "rw4m3": ["FTK_K1_RW=4", "FTK_K1_NSTAGE=3", "FTK_K1_MINB=3"],
    "vminb3": ["FTK_V_MINB=3"],
    "vminb4": ["FTK_V_MINB=4"],
    "vminb6": ["FTK_V_MINB=6"],
    "v3m3": ["FTK_V3_MINB=3"],
    "s3sp2": ["FTK_S3_SPLIT=2"],
    "gsr0": ["FTK_GATHER_SR=0"],
    "pair0": ["FTK_S3_PAIRSYNC=0"],
    "x3m1": ["FTK_X3_MINB=1"],
    "x3m4": ["FTK_X3_MINB=4"],
    "x3m6": ["FTK_X3_MINB=6"],
    "x3m8": ["FTK_X3_MINB=8"],
    "vminb8": ["FTK_V_MINB=8"],
    "jump2": ["FTK_LABEL_JUMP=2"],
    "jump4": ["FTK_LABEL_JUMP=4"],
    "xcount": ["FTK_X_COUNT=1"],
    "xru2": ["FTK_X_RUNROLL=2"],
    "s3r0": ["FTK_S3_REGION=0"],
    "s3cnt": ["FTK_S3_COUNT=1"],
    "s3sp1": ["FTK_S3_SPLIT=1"],
    "s3tp1": ["FTK_S3_TP=1"],
    "s3tp4": ["FTK_S3_TP=4"],
    "s3sp2": ["FTK_S3_SPLIT=2"],
    "s3noc": ["FTK_S3_NOCODES=1"],
    "s3noc8": ["FTK_S3_NOCODES=1", "FTK_S3_RW=8", "FTK_S3_MINB=1", "FTK_S3_NSTAGE=3"],
    "s3rw8": ["FTK_S3_RW=8", "FTK_S3_MINB=1", "FTK_S3_NSTAGE=3"],
    "s3st3": ["FTK_S3_NSTAGE=3", "FTK_S3_MINB=1"],
    "fprof": ["FTK_K1_PROF=1"],
    "fprof1": ["FTK_K1_PROF=1", "FTK_F_NXW=1"],
    "nxw1": ["FTK_F_NXW=1"],
    "nxw3": ["FTK_F_NXW=3"],
    "nxw4": ["FTK_F_NXW=4"],
    "xnopf": ["FTK_X_PREFETCH=0"],
}
names = sys.argv[1:] or list(VARIANTS)
for n in names:
    print(b.build_variant(n, VARIANTS[n]))
