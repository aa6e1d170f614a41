"""GPU box diagnostics of the bench's secondary legs on a config (e2e, stream, post, iso):
python tools/legs_check.py LEG [CONFIG] [NT]"""
import sys, time
sys.path.insert(0, '.')
import torch, ftk_inputs as fi, paper_2011_08697_b200 as ftk
leg = sys.argv[1]
cfg = fi.CONFIGS[sys.argv[2] if len(sys.argv) > 2 else 'C2']
nt = int(sys.argv[3]) if len(sys.argv) > 3 else None
f = cfg.make(nt).generate(device='cuda'); s = cfg.scale_log2
t = time.time()
if leg in ('iso', 'isonomesh'):
    out = ftk.iso_track(f, s, 0.5, return_buffers=True, mesh=leg == 'iso')
    torch.cuda.synchronize()
    print(leg, [tuple(o.shape) for o in out[:-1]], 'first call %.3f s' % (time.time() - t), flush=True)
    for _ in range(2):
        t = time.time()
        ftk.iso_track(f, s, 0.5, buffers=out[-1], mesh=leg == 'iso')
        torch.cuda.synchronize()
        print(leg, 'warm call %.3f s' % (time.time() - t), flush=True)
elif leg == 'e2e':
    rec, buf = ftk.track(f, s, return_buffers=True)
    host = f.cpu().pin_memory(); out = torch.empty(buf.capacity * ftk.RECORD_BYTES, dtype=torch.uint8).pin_memory()
    n = ftk.track_host(host, s, torch.empty_like(f), buf, out); print('e2e', n, time.time() - t, flush=True)
elif leg == 'stream':
    rec, buf = ftk.track(f, s, return_buffers=True)
    host = f.cpu().pin_memory(); sp = tuple(f.shape[1:])
    ws = torch.empty(ftk.Tracker.workspace_bytes(sp, f.dtype, s, buf.capacity, 64, False), dtype=torch.uint8, device='cuda')
    tr = ftk.Tracker(sp, f.dtype, s, buf.capacity, window=64, records=buf.records, workspace=ws)
    for p in range(host.shape[0]): tr.push(host[p])
    print('stream', tr.finish().shape, time.time() - t, flush=True)
elif leg == 'post':
    rec, buf = ftk.track(f, s, return_buffers=True); rec = rec.clone()
    tj = ftk.Trajectories(rec, buf, tuple(f.shape), f.dtype, s)
    print(tj.slice(f.shape[0] / 2 + 0.5).shape, tj.filter(f.shape[0] / 4, drop_loops=True).shape, flush=True)
    tj.smooth_types(2); torch.cuda.synchronize()
    print('post', time.time() - t, flush=True)
