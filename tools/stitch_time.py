"""Time the seam stitch of G virtual slabs of a config on one GPU: device path (pack + resolve +
relabel, what ftk_cp_track does with a communicator, minus the NCCL allgather) vs the host path."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import ftk_inputs as fi, paper_2011_08697_b200 as ftk

name = sys.argv[1] if len(sys.argv) > 1 else 'C2'
G = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = fi.CONFIGS[name]
w = cfg.make()
nt = cfg.shape[-1]
b = ftk.slab_bounds(nt, G)
cap = 1 << 17
stride = ftk.seam_block_size(cap)
blocks = torch.zeros(G * stride, dtype=torch.int64, device='cuda')
slabs = []
for r in range(G):
    ghost = r < G - 1
    sub = w.generate(t0=b[r], nt=b[r + 1] - b[r] + (1 if ghost else 0), device='cuda')
    rec, buf = ftk.track(sub, cfg.scale_log2, t0=b[r], nt_global=nt, ghost=ghost, return_buffers=True)
    slabs.append((sub, rec, buf, ghost, b[r]))
    A, B = ftk.stitch_export(sub, cfg.scale_log2, b[r], nt, ghost, buf)
    print(f'slab {r}: records {rec.shape[0]} A {len(A)} B {len(B)}')
for rep in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    for r, (sub, rec, buf, ghost, t0) in enumerate(slabs):
        ftk.seam_pack(sub, cfg.scale_log2, t0, nt, ghost, buf, blocks[r * stride:(r + 1) * stride], cap)
    for r, (sub, rec, buf, ghost, t0) in enumerate(slabs[:1]):
        ftk.seam_resolve(blocks, G, cap, rec)
    torch.cuda.synchronize(); td = (time.perf_counter() - t) * 1e3
    t = time.perf_counter()
    ex = [ftk.stitch_export(sub, cfg.scale_log2, t0, nt, ghost, buf) for (sub, rec, buf, ghost, t0) in slabs]
    GA = np.concatenate([e[0] for e in ex]); GB = np.concatenate([e[1] for e in ex])
    sub, rec, buf, ghost, t0 = slabs[0]
    old, new = ftk.stitch_resolve(GA, GB, np.concatenate([ex[0][0][:, 1], ex[0][1][:, 1]]))
    ftk.relabel(rec, old, new, buf)
    torch.cuda.synchronize(); th = (time.perf_counter() - t) * 1e3
    print(f'rep {rep}: device path {td:.3f} ms (pack all {G} + resolve one), host path {th:.3f} ms (export all + resolve + relabel one)')
