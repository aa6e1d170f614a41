import sys, time
sys.path.insert(0, '.')
import torch, ctypes, ftk_inputs as fi, paper_2011_08697_b200 as ftk
cfg = fi.CONFIGS['C2']; f = cfg.make().generate(device='cuda'); s = cfg.scale_log2
for cap in (70_000_000, 4_194_304):
    desc = ftk.make_desc(tuple(f.shape), f.dtype, s)
    b = ftk.Buffers.allocate(desc, cap, f.device)
    torch.cuda.synchronize()
    for rep in range(2):
        n_out = ctypes.c_int64(0)
        t = time.time()
        st = ftk.lib().ftk_iso_track(ctypes.byref(desc), ctypes.c_double(0.5), ctypes.c_void_p(f.data_ptr()),
                                    ctypes.c_void_p(b.records.data_ptr()), b.capacity, ctypes.byref(n_out),
                                    ctypes.c_void_p(b.workspace.data_ptr()), b.workspace.numel(), ctypes.c_void_p(0))
        torch.cuda.synchronize()
        print('cap', cap, 'status', st, 'n_out', n_out.value, '%.3f s' % (time.time() - t), flush=True)
