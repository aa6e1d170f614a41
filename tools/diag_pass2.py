import sys, os
sys.path.insert(0, '.')
import torch, ftk_inputs as fi, paper_2011_08697_b200 as ftk
for name in sys.argv[1:]:
    cfg = fi.CONFIGS[name]
    v = cfg.make().generate(device='cuda')
    vec = cfg.kind in ('gyre2d', 'abc3d')
    ftk.set_profiling(True)
    rec, buf = ftk.track(v, cfg.scale_log2, vector=vec, return_buffers=True)
    for i in range(2):
        rec = ftk.track(v, cfg.scale_log2, vector=vec, buffers=buf)
    ms, st = ftk.last_timings()
    print(name, 'pass2', ms[1], 'records', rec.shape[0])
