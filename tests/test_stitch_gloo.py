"""World-size-2 gloo test of the N > 1 host logic on CPU: each process takes one time slab (with a
ghost plane), derives its local labels and stitch lists from the ORACLE run on its slab as a domain
of its own (no GPU), exchanges the lists with torch.distributed all_gather_object, resolves them with
the library's host resolver (ftk_stitch_resolve) and relabels; the result must equal the
single-domain oracle labels on every owned face."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _slab_labels(field, s, t0, t1, ghost, T, plane):
    """oracle on planes [t0, t1 (+ ghost)] as its own domain; ids shifted to global t"""
    import oracle
    sub = np.ascontiguousarray(field[t0: t1 + (1 if ghost else 0)])
    rec, _, _ = oracle.track(sub, s)
    shift = t0 * plane * T
    fid = rec["face_id"] + shift
    lab = rec["label"] + shift
    t_of = fid // T // plane
    ordinal = (rec["flags"] & 1) != 0
    own = t_of < t1
    A = np.stack([fid[~own], lab[~own]], 1) if ghost else np.zeros((0, 2), np.int64)
    B = np.stack([fid[own & ordinal & (t_of == t0)], lab[own & ordinal & (t_of == t0)]], 1) if t0 > 0 \
        else np.zeros((0, 2), np.int64)
    return fid[own], lab[own], A, B


def _worker(rank, world, port, q, nt, shape3):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import ftk_inputs as fi
        import paper_2011_08697_b200 as ftk
        import oracle
        w = fi.Woven(shape3[0], shape3[1], nt, sigma=0.02)
        f = w.generate().numpy()
        T, plane = 12, shape3[0] * shape3[1]
        b = ftk.slab_bounds(nt, world)
        fid, lab, A, B = _slab_labels(f, 26, b[rank], b[rank + 1], rank < world - 1, T, plane)
        gathered = [None] * world
        dist.all_gather_object(gathered, (A, B))
        GA = np.concatenate([g[0] for g in gathered])
        GB = np.concatenate([g[1] for g in gathered])
        old, new = ftk.stitch_resolve(GA, GB, np.concatenate([A[:, 1], B[:, 1]]))
        m = dict(zip(old.tolist(), new.tolist()))
        lab2 = np.array([m.get(int(l), int(l)) for l in lab], np.int64)
        ref, _, _ = oracle.track(f, 26)
        refmap = dict(zip(ref["face_id"].tolist(), ref["label"].tolist()))
        ok = all(refmap[int(a)] == int(l) for a, l in zip(fid, lab2)) and len(fid) > 0
        owned_ref = sum(1 for x in ref["face_id"] if b[rank] <= x // T // plane < b[rank + 1])
        q.put((rank, ok, len(fid) == owned_ref, len(A), len(B)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_two_slabs_match_single_domain(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, 21, (40, 36))) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    res = sorted(q.get(timeout=5) for _ in range(world))
    for rank, ok, complete, nA, nB in res:
        assert ok and complete, res
    assert res[0][3] > 0 and res[1][4] > 0  # the seam actually carries trajectories
