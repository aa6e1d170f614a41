"""Profiling driver: one warm-up + N measured track calls on a config (for ncu / nsys-less timing)."""
import sys, time
sys.path.insert(0, '.')
import torch
import ftk_inputs as fi, paper_2011_08697_b200 as ftk

name = sys.argv[1] if len(sys.argv) > 1 else 'C2'
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = fi.CONFIGS[name]
f = cfg.make().generate(device='cuda')
vec = cfg.kind in ('gyre2d', 'abc3d')
ftk.set_profiling(True)
rec, buf = ftk.track(f, cfg.scale_log2, return_buffers=True, vector=vec)
for i in range(reps):
    rec = ftk.track(f, cfg.scale_log2, buffers=buf, vector=vec)
    ms, st = ftk.last_timings()
    km = ftk.last_kernel_timings()
    print(f'{name} rep {i}: k1 {ms[0]:.3f} ms (k1a {km[0]:.3f} k1b {km[1]:.3f}) pass2 {ms[1]:.3f} ms call {ms[3]:.3f} ms faces {st[0]} survivors {st[1]} punctured {st[2]}')
torch.cuda.synchronize()
if '--counters' in sys.argv:
    c = buf.workspace[:256].view(torch.int64).cpu().tolist()
    print('counters[16..30]:', c[16:30])
