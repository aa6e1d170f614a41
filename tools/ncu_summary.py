"""Summarise ncu outputs into profiles/: the launch list (per-kernel device time shares) and the
key metrics of one --set full capture of K1.  Usage:
  python tools/ncu_summary.py <launches.csv> <k1.ncu-rep> <tag> [config]"""
import collections, csv, json, os, subprocess, sys

launches, rep, tag = sys.argv[1], sys.argv[2], sys.argv[3]
config = sys.argv[4] if len(sys.argv) > 4 else "C2"
out_dir = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")
os.makedirs(out_dir, exist_ok=True)

rows = list(csv.reader(open(launches)))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
per = collections.defaultdict(list)
for r in rows[start + 1:]:
    if len(r) > vi:
        per[r[ki]].append(float(r[vi].replace(",", "")) / 1000.0)
ours = {k: v for k, v in per.items() if any(s in k for s in ("k2d::", "trk::", "k3d::", "ftk::"))}
tot = sum(sum(v) for v in ours.values())
lines = [f"# ncu launch list ({tag}, {config}): gpu__time_duration.sum, --clock-control none, cold-cache serialised",
         "# kernel | launches | mean us | share of our kernels' time"]
for k, v in sorted(ours.items(), key=lambda kv: -sum(kv[1])):
    lines.append(f"{k[:70]} | {len(v)} | {sum(v)/len(v):.1f} | {100*sum(v)/tot:.1f}%")
open(os.path.join(out_dir, f"launches_{tag}.txt"), "w").write("\n".join(lines) + "\n")
print("\n".join(lines))

raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
d = dict(zip(r[0], r[2]))
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "lts__t_sectors_srcunit_tex_op_read.sum"]
units = dict(zip(r[0], r[1]))
summary = {k: (d.get(k), units.get(k)) for k in keys if k in d}
stalls = sorted(((k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v or 0)) for k, v in d.items()
                 if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")),
                key=lambda kv: -kv[1])
tot_s = sum(v for _, v in stalls) or 1
summary["stall_samples_top"] = [(k, round(100 * v / tot_s, 1)) for k, v in stalls[:8]]
json.dump(summary, open(os.path.join(out_dir, f"k1_ncu_{tag}.json"), "w"), indent=1)
print(json.dumps(summary, indent=1))

def num(x):
    return float(str(x).replace(",", ""))

# dram bytes per launch for bench.py's roofline.traffic (ncu reports in the unit it picked)
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rd = num(d["dram__bytes_read.sum"]) * scale.get(units["dram__bytes_read.sum"], 1)
wr = num(d["dram__bytes_write.sum"]) * scale.get(units["dram__bytes_write.sum"], 1)
tp = os.path.join(out_dir, "k1_traffic.json")
t = json.load(open(tp)) if os.path.exists(tp) else {}
t[config] = rd + wr
json.dump(t, open(tp, "w"), indent=1)
print("traffic bytes per K1 launch:", rd + wr)
