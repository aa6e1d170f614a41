"""Per-step time of repeated track calls with and without the CUDA-graph replay (FTK_DEBUG_NO_GRAPH):
CUDA events around K calls on the current stream, as bench.py times its steps.
usage: python tools/graph_time.py [CONFIG] [K]"""
import sys
sys.path.insert(0, '.')
import torch
import ftk_inputs as fi, paper_2011_08697_b200 as ftk

name = sys.argv[1] if len(sys.argv) > 1 else 'C2'
K = int(sys.argv[2]) if len(sys.argv) > 2 else 100
cfg = fi.CONFIGS[name]
f = cfg.make().generate(device='cuda')
vec = cfg.kind in ('gyre2d', 'abc3d')
rec, buf = ftk.track(f, cfg.scale_log2, return_buffers=True, vector=vec)
s = torch.cuda.current_stream()
for flags, label in ((ftk.DEBUG_NO_GRAPH, 'plain launches'), (0, 'graph replay'), (ftk.DEBUG_NO_GRAPH, 'plain launches'),
                     (0, 'graph replay')):
    ftk.set_debug(flags)
    for _ in range(5):
        ftk.track(f, cfg.scale_log2, buffers=buf, vector=vec)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(K):
        ftk.track(f, cfg.scale_log2, buffers=buf, vector=vec)
    b.record(s)
    torch.cuda.synchronize()
    print(f'{name} {label}: {a.elapsed_time(b) / K:.4f} ms/step')
ftk.set_debug(0)
