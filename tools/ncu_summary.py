"""Summarise ncu outputs into profiles/ (round tag):
  launches_<tag>.txt      -- per-kernel device time shares from a --metrics gpu__time_duration.sum launch list
  ncu_<tag>_<kernel>.json -- key metrics + stall breakdown of each kernel in a --set full capture
  ncu_traffic.json        -- {config: {kernel: dram read+write bytes per launch}} (read by bench.py)
usage: python tools/ncu_summary.py <launches.csv> <full.ncu-rep> <tag> [config]"""
import collections, csv, json, os, subprocess, sys

launches, rep, tag = sys.argv[1], sys.argv[2], sys.argv[3]
config = sys.argv[4] if len(sys.argv) > 4 else "C2"
out_dir = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")
os.makedirs(out_dir, exist_ok=True)


def num(v):
    try:
        return float(v.replace(",", ""))
    except (ValueError, AttributeError):
        return None


rows = list(csv.reader(open(launches)))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
per = collections.defaultdict(list)
for r in rows[start + 1:]:
    if len(r) > vi and num(r[vi]) is not None:
        per[r[ki]].append(num(r[vi]) / 1000.0)
# the step's kernels (the bench's post-processing leg -- k_verify adjacency, k_post_* -- is not part of it)
ours = {k: v for k, v in per.items() if any(s in k for s in ("k2d::", "trk::", "k3d::", "ftk::", "k_"))
        and "k_verify" not in k and "k_post" not in k}
tot = sum(sum(v) for v in ours.values())
lines = [f"# ncu launch list ({tag}, {config}): gpu__time_duration.sum, --clock-control none, cold-cache serialised",
         "# kernel | launches | mean us | share of our kernels' time"]
for k, v in sorted(ours.items(), key=lambda kv: -sum(kv[1])):
    lines.append(f"{k[:70]} | {len(v)} | {sum(v)/len(v):.1f} | {100*sum(v)/tot:.1f}%")
open(os.path.join(out_dir, f"launches_{tag}.txt"), "w").write("\n".join(lines) + "\n")
print("\n".join(lines))

raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
hdr, units = r[0], r[1]
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_sectors_srcunit_tex_op_read.sum"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
tp = os.path.join(out_dir, "ncu_traffic.json")
traffic = json.load(open(tp)) if os.path.exists(tp) else {}
for row in r[2:]:
    d = dict(zip(hdr, row))
    u = dict(zip(hdr, units))
    name = d.get("Kernel Name", "?")
    short = name.split("(")[0].split("::")[-1].split("<")[0].strip().split()[-1]
    out = {"kernel": name, "config": config, "tag": tag}
    for k in KEYS:
        if k in d:
            out[k] = [d[k], u.get(k, "")]
    st = []
    for h in hdr:
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            v = num(d[h])
            if v:
                st.append((v, h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
    tot_s = sum(v for v, _ in st) or 1
    out["stall_samples_top"] = [[n, round(100 * v / tot_s, 1)] for v, n in sorted(st, reverse=True)[:10]]
    try:
        b = num(d["dram__bytes_read.sum"]) * SCALE[u["dram__bytes_read.sum"]] + \
            num(d["dram__bytes_write.sum"]) * SCALE[u["dram__bytes_write.sum"]]
        traffic.setdefault(config, {})[short] = b
        out["dram_bytes_per_launch"] = b
    except (KeyError, TypeError):
        pass
    json.dump(out, open(os.path.join(out_dir, f"ncu_{tag}_{short}.json"), "w"), indent=1)
    print("wrote", f"ncu_{tag}_{short}.json", out.get("dram_bytes_per_launch"))
json.dump(traffic, open(tp, "w"), indent=1)
