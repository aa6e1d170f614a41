#!/usr/bin/env python
"""Benchmark of the FTK critical-point tracking hot path on B200 (bench contract: ONE JSON line).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

A step is one full `track` call (all SURVEY.md 8(a) rows: closed-form mesh, fused quantize/gradient
prefilter, exact SoS test, location/type, compaction, link, union-find, labels) over one batch of
synthetic input already resident in HBM.  Metric (BASELINE.json): spacetime faces tested per second
(every face gets a definitive classification), plus the K1 extraction kernel's fraction of the
measured HBM roofline.

N = 1: workload C2 (2D woven 1024 x 1024 x 256, BASELINE.json configs[1]).
N > 1 (default --scaling weak): every rank owns a C2-sized time slab (256 timesteps + one ghost plane)
of a global woven field with 256*N timesteps; trajectories are stitched across slabs (NCCL).
--scaling strong: the configuration's whole time axis (e.g. --config C4, 4096^2 x 512, the north_star
strong-scaling target) split into N contiguous slabs of nt/N timesteps + one ghost plane; N = 1 tracks
the whole field on one GPU.  The driver computes the scaling efficiency from the per-N values.

--impl reference: the CPU oracle (oracle/, plain C + OpenMP, never tuned) on this box's host cores,
same metric and config, each step a bounded sample of the workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "spacetime faces tested/sec"
UNIT = "faces/s"


def _dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """Samples SM clocks and throttle reasons with NVML during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.ok = [], 0, False
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.0005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml_unavailable"]}
        names = [n for b, n in self.REASONS.items() if self.reasons & b and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz, "reasons": names,
                "samples": len(self.samples)}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def _ncu_traffic(config_name: str, kernel: str = "k_scan2d"):
    """dram read + write bytes per launch of `kernel` from the committed ncu --set full summary
    (profiles/ncu_traffic.json: {config: {kernel: bytes}}), if present"""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(config_name, {}).get(kernel)
    except Exception:
        return None


def cpu_baseline(cfg, seconds_budget: float = 20.0):
    """The oracle, as it stands, on the host cores: track on a bounded sample of the workload
    (full spatial plane, first nt_s timesteps as its own domain).  Returns a dict."""
    import oracle
    import ftk_inputs as fi
    import paper_2011_08697_b200 as ftk

    spatial = cfg.shape[:-1]
    nt_s = 3
    w = cfg.make()
    if len(spatial) == 3:
        # 3D: a 64^3 block of the same field kind as its own domain keeps the oracle within ~20 s
        w = fi.ABCFlow(64, 64, 64, nt_s, scale_log2=cfg.scale_log2) if cfg.kind == "abc3d" else \
            fi.Woven(64, 64, nt_s, nz=64, scale_log2=cfg.scale_log2) if cfg.kind == "woven3d" else \
            fi.MovingExtremum((64, 64, 64), nt_s, c0=(30.0, 31.0, 32.0), v=(0.25, 0.125, -0.0625),
                              scale_log2=cfg.scale_log2)
        spatial = (64, 64, 64)
    f = w.generate(nt=nt_s).numpy()
    cores = os.cpu_count() or 1
    t = time.perf_counter()
    rec, nf, info = oracle.track(f, cfg.scale_log2, nthreads=cores, vector=cfg.kind in ("gyre2d", "abc3d"))
    dt = time.perf_counter() - t
    return {"value": nf / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"oracle track (plain C, OpenMP {cores} threads) on {'x'.join(map(str, spatial))}x{nt_s} "
                      f"timesteps of a {cfg.name}-kind field as its own domain: {nf} faces in {dt:.2f} s "
                      f"({dt * cores:.0f} core-seconds)"}


def run_reference(args):
    """--impl reference: the oracle on the host cores, same metric/config, bounded samples."""
    rank, world, _ = _dist_env()
    if rank != 0:
        return 0
    import oracle
    import ftk_inputs as fi

    cfg = fi.CONFIGS[args.config]
    spatial = cfg.shape[:-1]
    ny = spatial[-1]           # extent of the sliced axis (y in 2D, z in 3D; the field is [t][z][y][x])
    cores = os.cpu_count() or 1
    w = cfg.make()
    # per-step sample: a band of rows (2D) / slices (3D) x 2 timesteps of the workload's field, sized
    # so the whole run ends in about two minutes
    total_budget = 120.0
    per_step = total_budget / max(1, args.steps + args.warmup)
    rows = 16
    f_full = w.generate(nt=2).numpy()
    while True:
        f = f_full[:, :rows, :].copy()
        t = time.perf_counter()
        rec, nf, info = oracle.track(f, cfg.scale_log2, nthreads=cores, vector=cfg.kind in ("gyre2d", "abc3d"))
        dt = time.perf_counter() - t
        if dt > per_step * 0.5 or rows >= ny:
            break
        rows = min(ny, rows * 2)
    times = []
    for i in range(args.warmup + args.steps):
        t = time.perf_counter()
        rec, nf, info = oracle.track(f, cfg.scale_log2, nthreads=cores, vector=cfg.kind in ("gyre2d", "abc3d"))
        dt = time.perf_counter() - t
        if i >= args.warmup:
            times.append(dt)
    ms = 1000.0 * sum(times) / len(times)
    value = nf / (ms / 1000.0)
    band = "x".join(map(str, list(spatial[:-1]) + [rows]))
    sample = f"oracle track on {band}x2 of {cfg.name} per step ({nf} faces), {cores} threads"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": f"{cfg.name}: {cfg.desc}", "sample": sample},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist

    import ftk_inputs as fi
    import paper_2011_08697_b200 as ftk

    rank, world, local = _dist_env()
    if args.gpus > 1 or world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", init_method="env://")
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)
    ftk.lib()

    cfg = fi.CONFIGS[args.config]
    spatial, nt = cfg.shape[:-1], cfg.shape[-1]
    vec = cfg.kind in ("gyre2d", "abc3d")  # vector fields (FTK_VECTOR_FIELD), SURVEY.md 8(f) NEXT row 2
    w = cfg.make()
    if args.scaling == "strong":  # the config's time axis split into world slabs (+ one ghost plane)
        b = ftk.slab_bounds(nt, world)
        nt_global, t0, ghost = nt, b[rank], rank < world - 1
        nbuf = b[rank + 1] - b[rank] + (1 if ghost else 0)
    elif world > 1:  # weak: a slab of the config's size per rank
        nt_global = nt * world
        w.nt = nt_global
        t0 = rank * nt
        ghost = rank < world - 1
        nbuf = nt + (1 if ghost else 0)
    else:
        nt_global, t0, ghost, nbuf = nt, 0, False, nt
    field = w.generate(t0=t0, nt=nbuf, device=dev)
    desc = ftk.make_desc(tuple(field.shape), field.dtype, cfg.scale_log2, t0=t0, nt_global=nt_global, ghost=ghost,
                         vector=vec)
    faces = ftk.num_faces(desc)
    # multi-GPU: trajectories crossing slab seams are stitched inside ftk_cp_track (NCCL allgather of
    # the seam pairs, host union, device relabel)
    comm = ftk.Comm(rank, world, device=dev) if world > 1 else None
    cptr = comm.ptr if comm is not None else None

    stream = torch.cuda.current_stream(dev)
    ftk.set_profiling(False)
    rec, buf = ftk.track(field, cfg.scale_log2, t0=t0, nt_global=nt_global, ghost=ghost, comm=cptr, return_buffers=True,
                         vector=vec)
    n_punct = rec.shape[0]
    # warmup
    for _ in range(args.warmup):
        ftk.track(field, cfg.scale_log2, t0=t0, nt_global=nt_global, ghost=ghost, buffers=buf, comm=cptr, vector=vec)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index or 0) as clk:
        start.record(stream)
        for _ in range(args.steps):
            ftk.track(field, cfg.scale_log2, t0=t0, nt_global=nt_global, ghost=ghost, buffers=buf, comm=cptr, vector=vec)
        stop.record(stream)
        torch.cuda.synchronize(dev)
    ms_total = start.elapsed_time(stop)
    # per-kernel split (CUDA events recorded by the library around each kernel on the launch stream),
    # in a separate profiled pass so the events do not sit inside the headline timing
    k1_ms, p2_ms, st_ms, ka_ms, kb_ms = [], [], [], [], []
    ftk.set_profiling(True)
    for _ in range(max(3, min(args.steps, 30))):
        ftk.track(field, cfg.scale_log2, t0=t0, nt_global=nt_global, ghost=ghost, buffers=buf, comm=cptr, vector=vec)
        ms4, st3 = ftk.last_timings()
        km = ftk.last_kernel_timings()
        ka_ms.append(km[0])
        kb_ms.append(km[1])
        k1_ms.append(ms4[0])
        p2_ms.append(ms4[1])
        st_ms.append(ms4[2])
    ftk.set_profiling(False)
    if clk.ok and len(clk.samples) < 5:
        # short timed regions: keep the GPU busy with the same step and sample again
        with ClockSampler(dev.index or 0) as clk2:
            t_end = time.perf_counter() + 0.3
            while time.perf_counter() < t_end:
                ftk.track(field, cfg.scale_log2, t0=t0, nt_global=nt_global, ghost=ghost, buffers=buf, comm=cptr, vector=vec)
            torch.cuda.synchronize(dev)
        clk.samples += clk2.samples
        clk.reasons |= clk2.reasons
    if world > 1:
        t = torch.tensor([ms_total], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
        ft = torch.tensor([faces], device=dev, dtype=torch.float64)
        dist.all_reduce(ft)
        total_faces = float(ft.item())
    else:
        total_faces = float(faces)
    ms_step = ms_total / args.steps
    value = total_faces / (ms_step / 1000.0)

    # roofline of the extraction pass north_star names: algorithmic bytes = the field
    # read once + 56 B per punctured face written (halo re-reads, ghost planes and workspace traffic --
    # the survivor windows K1a hands to K1b, face ids, union-find parents, edges -- are not
    # algorithmic); time = the whole pass, K1a scan + K1b exact (+ k_expand2d on the 2D vector path),
    # from CUDA events the library records on the launch stream; K1a and K1b are broken out beside it
    # with their own ncu dram traffic, and the whole step's fraction on the same bytes
    esz = field.element_size()
    k1_avg = sum(k1_ms) / len(k1_ms)
    ka_avg = sum(ka_ms) / len(ka_ms)
    kb_avg = sum(kb_ms) / len(kb_ms)
    _, st3 = ftk.last_timings()
    n_surv = st3[1]
    d3 = len(spatial) == 3
    field_bytes = field.numel() * esz
    rec_bytes = n_punct * ftk.RECORD_BYTES
    alg_bytes = field_bytes + rec_bytes
    achieved = alg_bytes / (k1_avg / 1000.0) / 1e9
    peak, peak_src = _peaks()
    if d3:
        kscan, kexact = ("k_scanvec3d", "k_exact3d") if vec else ("k_scan3d", "k_exact3d")
    else:
        kscan, kexact = ("k_scanvec2d", "k_exactvec2d") if vec else ("k_scan2d", "k_exact2d")
    t_scan, t_exact = _ncu_traffic(cfg.name, kscan), _ncu_traffic(cfg.name, kexact)
    traffic = t_scan + t_exact if t_scan is not None and t_exact is not None else None

    # end to end through the C-ABI from pinned host memory (H2D + D2H inside the timed region)
    e2e = None
    if world > 1 and not args.no_e2e:
        # every rank: its slab from pinned host memory, track with the stitch, records back to the host;
        # CUDA events on the launch stream, max over ranks
        host = field.cpu().pin_memory()
        stage = torch.empty_like(field)
        times, nrec = [], 0
        for i in range(max(3, min(args.steps, 20)) + 1):
            dist.barrier()
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            stage.copy_(host, non_blocking=True)
            rec_e = ftk.track(stage, cfg.scale_log2, t0=t0, nt_global=nt_global, ghost=ghost, buffers=buf, comm=cptr,
                              vector=vec)
            out = rec_e.cpu()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            nrec = out.shape[0]
            if i:
                times.append(e0.elapsed_time(e1))
        t = torch.tensor([sum(times) / len(times)], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t.item())
        e2e = {"value": total_faces / (e_ms / 1000.0), "unit": UNIT, "ms_per_step": e_ms,
               "h2d_bytes_per_step": field.numel() * esz, "d2h_bytes_per_step": nrec * ftk.RECORD_BYTES,
               "per": "rank (max over ranks); bytes of rank 0"}
        del host, stage
    if world == 1 and not args.no_e2e:
        host = field.cpu().pin_memory()
        out_host = torch.empty(buf.capacity * ftk.RECORD_BYTES, dtype=torch.uint8).pin_memory()
        stage = torch.empty_like(field)
        n = ftk.track_host(host, cfg.scale_log2, stage, buf, out_host, vector=vec)  # warm
        e_steps = max(3, min(args.steps, 20))
        torch.cuda.synchronize(dev)
        t = time.perf_counter()
        for _ in range(e_steps):
            n = ftk.track_host(host, cfg.scale_log2, stage, buf, out_host, vector=vec)
        e_ms = (time.perf_counter() - t) * 1000.0 / e_steps
        e2e = {"value": faces / (e_ms / 1000.0), "unit": UNIT, "ms_per_step": e_ms,
               "h2d_bytes_per_step": field.numel() * esz, "d2h_bytes_per_step": n * ftk.RECORD_BYTES + 64}

    # streaming ingestion: every plane pushed from pinned host memory, one timestep at a
    # time, windows of 64 (+ ghost) resident on the device; pass 2 at the end -- wall clock around
    # whole streams (H2D inside), records identical to track()
    stream_line = None
    if world == 1 and not args.no_e2e and not args.no_stream:
        window = 64
        host = field.cpu().pin_memory()
        planes = [host[t] for t in range(host.shape[0])]
        sp = tuple(field.shape[1:])
        ws = torch.empty(ftk.Tracker.workspace_bytes(sp, field.dtype, cfg.scale_log2, buf.capacity, window, vec),
                         dtype=torch.uint8, device=dev)

        def one_stream():
            tr = ftk.Tracker(sp, field.dtype, cfg.scale_log2, buf.capacity, window=window,
                             records=buf.records, workspace=ws, vector=vec)
            for p in planes:
                tr.push(p)
            return tr.finish().shape[0]

        n_s = one_stream()
        s_steps = max(3, min(args.steps, 10))
        torch.cuda.synchronize(dev)
        t = time.perf_counter()
        for _ in range(s_steps):
            n_s = one_stream()
        s_ms = (time.perf_counter() - t) * 1000.0 / s_steps
        stream_line = {"value": faces / (s_ms / 1000.0), "unit": UNIT, "ms_per_step": s_ms, "window": window,
                       "resident_planes": window + 1, "records": int(n_s),
                       "h2d_bytes_per_step": field.numel() * esz, "timing": "wall clock, synchronised"}
        del ws, host, planes

    # trajectory post-processing over this step's records: adjacency, a slice,
    # a duration filter, simplification in time (tau = 2 timesteps) and type smoothing, each synchronous;
    # wall clock per operation
    post_line = None
    if world == 1 and not args.no_stream and not args.no_e2e and not d3:
        rec_p, buf_p = ftk.track(field, cfg.scale_log2, buffers=buf, vector=vec, return_buffers=True)
        rec_p = rec_p.clone()
        tp = {}
        torch.cuda.synchronize(dev)
        t = time.perf_counter()
        tj = ftk.Trajectories(rec_p, buf_p, tuple(field.shape), field.dtype, cfg.scale_log2, vector=vec)
        tp["adjacency_ms"] = (time.perf_counter() - t) * 1000.0
        t = time.perf_counter()
        n_slice = tj.slice(nt_global / 2 + 0.5).shape[0]
        tp["slice_ms"] = (time.perf_counter() - t) * 1000.0
        t = time.perf_counter()
        n_filt = tj.filter(nt_global / 4, drop_loops=True).shape[0]
        tp["filter_ms"] = (time.perf_counter() - t) * 1000.0
        t = time.perf_counter()
        tj.simplify_types(2.0)
        torch.cuda.synchronize(dev)
        tp["simplify_ms"] = (time.perf_counter() - t) * 1000.0
        t = time.perf_counter()
        tj.smooth_types(2)
        torch.cuda.synchronize(dev)
        tp["smooth_ms"] = (time.perf_counter() - t) * 1000.0
        post_line = {**tp, "records": int(rec_p.shape[0]), "slice_points": int(n_slice), "filtered_records": int(n_filt),
                     "timing": "wall clock per synchronous call, after one warm track"}
        del tj, rec_p

    # isovolume tracking on the same field: spacetime edges
    # tested per second by ftk_iso_track (isovalue 0.5 in 2D; 1.9 near the maxima of the 3D fields, whose
    # 0.5-level isovolume would not fit next to the field), CUDA events around the synchronous call
    iso_line = None
    if world == 1 and not args.no_e2e and not vec and field.numel() * field.element_size() > (8 << 30):
        # C4: the 0.5-level isovolume of the 34 GB woven field holds ~2e9 records (112 GB), which do not
        # fit next to the field
        iso_line = {"skipped": "isovolume records of a field > 8 GiB do not fit next to it in HBM"}
    elif world == 1 and not args.no_e2e and not vec:
        iso_val = 1.9 if d3 else 0.5
        rec_i, el_i, buf_i = ftk.iso_track(field, cfg.scale_log2, iso_val, return_buffers=True, mesh=True)
        ext = list(spatial) + [nt_global]
        n_edges = 0
        for m in range(1, 1 << len(ext)):
            k = 1
            for a, n in enumerate(ext):
                k *= n - ((m >> a) & 1)
            n_edges += k
        i_ms = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ftk.iso_track(field, cfg.scale_log2, iso_val, buffers=buf_i, mesh=True)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            i_ms.append(e0.elapsed_time(e1))
        i_best = min(i_ms)
        iso_line = {"isovalue": iso_val, "edges_per_step": n_edges, "value": n_edges / (i_best / 1000.0),
                    "unit": "spacetime edges/s", "ms": i_best, "records": int(rec_i.shape[0]),
                    "simplices": int(el_i.shape[0]), "simplex": "tetrahedra" if d3 else "triangles",
                    "components": int(len(torch.unique(rec_i[:, 1]))) if rec_i.shape[0] else 0,
                    "timing": "CUDA events around ftk_iso_track_mesh (edge + cell pass with the mesh + pass 2), best of 5"}
        del rec_i, el_i, buf_i

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": f"{cfg.name}: {cfg.desc}" + (
                       f", {world} time slabs of {nt} + ghost" if world > 1 and args.scaling == "weak" else
                       f", strong scaling: {nt} timesteps in {world} slab(s) of ~{nt // world} + ghost"
                       if args.scaling == "strong" else ""),
                   "grid": [*spatial, nt_global], "faces_per_step": int(total_faces),
                   "punctured_per_step": int(n_punct), "input": f"{field.dtype}".replace("torch.", ""),
                   "arith": "exact int64/int128 predicates, fixed-order f64 location/type, f32 prefilter",
                   "l2": "input (%.2f GB) larger than L2 (126 MB); no flush" % (field.numel() * esz / 1e9),
                   "k1_ms": k1_avg, "k1a_scan_ms": ka_avg, "k1b_exact_ms": kb_avg,
                   "survivors_per_step": int(n_surv), "pass2_ms": sum(p2_ms) / len(p2_ms),
                   **({"stitch_ms": sum(st_ms) / len(st_ms)} if world > 1 else {})},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "kernel": f"extraction pass: {kscan} (K1a scan) + {kexact} (K1b exact)",
                     "alg_bytes_per_launch": alg_bytes,
                     "alg_bytes": "SURVEY.md 8(d): field read once (%d B) + 56 B x %d punctured faces" % (
                         field_bytes, n_punct),
                     "ms": k1_avg, "share_of_step": k1_avg / ms_step,
                     "step_frac": alg_bytes / (ms_step / 1000.0) / 1e9 / peak,
                     kscan: {"ms": ka_avg, "share_of_step": ka_avg / ms_step, "alg_bytes": field_bytes,
                             "frac": field_bytes / (ka_avg / 1000.0) / 1e9 / peak, "traffic": t_scan},
                     kexact: {"ms": kb_avg, "share_of_step": kb_avg / ms_step, "alg_bytes": rec_bytes,
                              "frac": rec_bytes / (kb_avg / 1000.0) / 1e9 / peak if kb_avg > 0 else None,
                              "traffic": t_exact}},
        "clocks": clk.summary(),
        "e2e": e2e,
        "stream": stream_line,
        "post": post_line,
        "iso": iso_line,
        # K1a + K1b (+ k_expand2d in 2D) + k_clear + k_hash_insert + k_edges + k_root + k_label (one CUDA
        # graph per step; the ncu launch list shows them); time slabs add k_export and the device seam
        # path (k_seam_pack, _clear, _insert, _union, _relabel)
        "gpu_launches": ((7 if d3 else 8) + (6 if world > 1 else 0)) * args.steps,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg)
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        comm.close()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-stream", action="store_true")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N > 1: weak = a config-sized slab per rank; strong = the config's time axis split")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
