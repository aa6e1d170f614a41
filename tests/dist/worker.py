"""torchrun worker for tests/dist (one process per GPU): time slabs tracked with a real NCCL
communicator (ftk.Comm, ftk_cp_track stitching over NVLink) must give exactly the single-GPU records and
global labels; a failure on one slab must surface as the same error on every rank
(include/ftk_cp.h: the failure code travels in the seam exchange).

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 --master-port P \\
        tests/dist/worker.py OUT_DIR
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import ftk_inputs as fi  # noqa: E402
import paper_2011_08697_b200 as ftk  # noqa: E402


def slab(field, rank, world):
    nt = field.shape[0]
    b = ftk.slab_bounds(nt, world)
    ghost = rank < world - 1
    return field[b[rank]: b[rank + 1] + (1 if ghost else 0)].contiguous(), b[rank], nt, ghost


def main():
    out_dir = sys.argv[1]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", init_method="env://")
    ftk.lib()
    comm = ftk.Comm(rank, world, device=dev)
    ok = True
    cases = [("woven2d", fi.Woven(96, 80, 8 * world + 5, sigma=0.02).generate()),
             ("woven3d", fi.Woven(23, 21, 3 * world + 4, L=15.0, sigma=0.02, nz=19).generate()),
             ("c2_crop", fi.CONFIGS["C2"].make(nt=16 * world).generate()[:, 256:512, 384:768].contiguous())]
    for name, f in cases:
        sub, t0, nt, ghost = slab(f, rank, world)
        for rep in range(2):  # the second call runs on the communicator's warm seam blocks
            rec = ftk.to_numpy(ftk.track(sub.to(dev), 26, t0=t0, nt_global=nt, ghost=ghost, comm=comm.ptr))
        np.save(os.path.join(out_dir, f"{name}_rank{rank}.npy"), rec)
        if rank == 0:
            single = ftk.to_numpy(ftk.track(f.to(dev), 26))
            np.save(os.path.join(out_dir, f"{name}_single.npy"), single)
    # a non-finite value in one slab: every rank must report FTK_ERR_RANGE (no rank left in NCCL)
    f = fi.Woven(64, 48, 4 * world + 3, sigma=0.02).generate()
    sub, t0, nt, ghost = slab(f, rank, world)
    if rank == world - 1:
        sub[1, 5, 7] = float("nan")
    status = 0
    try:
        ftk.track(sub.to(dev), 26, t0=t0, nt_global=nt, ghost=ghost, comm=comm.ptr)
    except ftk.FtkError as e:
        status = e.status
    st = torch.tensor([status], device=dev)
    allst = [torch.zeros_like(st) for _ in range(world)]
    dist.all_gather(allst, st)
    with open(os.path.join(out_dir, f"status_rank{rank}.txt"), "w") as fh:
        fh.write(" ".join(str(int(x.item())) for x in allst))
    # the communicator still works after the failed call
    sub, t0, nt, ghost = slab(fi.Woven(64, 48, 4 * world + 3, sigma=0.02).generate(), rank, world)
    ftk.track(sub.to(dev), 26, t0=t0, nt_global=nt, ghost=ghost, comm=comm.ptr)
    dist.barrier()
    comm.close()
    dist.destroy_process_group()
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
