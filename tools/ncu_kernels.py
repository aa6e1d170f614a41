"""Key metrics per captured kernel of an ncu --set full report.  usage: ncu_kernels.py rep.ncu-rep"""
import csv, subprocess, sys
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
hdr = r[0]
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "lts__t_sectors_op_atom.sum", "lts__t_sectors_op_red.sum", "l1tex__t_bytes_pipe_lsu_mem_global_op_ld.sum",
        "lts__t_bytes.sum"]
stall = [h for h in hdr if h.startswith("smsp__average_warp_latency_issue_stalled") or
         (h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"))]
for row in r[2:]:
    d = dict(zip(hdr, row))
    print("==", d.get("Kernel Name", "?")[:80])
    for k in KEYS:
        if k in d:
            print(f"   {k:60s} {d[k]} {r[1][hdr.index(k)]}")
    ss = []
    for h in stall:
        try:
            ss.append((float(d[h].replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except (ValueError, KeyError):
            pass
    tot = sum(v for v, _ in ss) or 1
    print("   stalls:", ", ".join(f"{n} {100*v/tot:.0f}%" for v, n in sorted(ss, reverse=True)[:8]))
