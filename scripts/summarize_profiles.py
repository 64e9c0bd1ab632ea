"""Summaries under profiles/ from a gpu_round.sh run: launch list shares, ncu
full-capture key metrics and stall reasons, traffic per launch.
Usage: python scripts/summarize_profiles.py <tag> <workload-name>"""
import collections
import csv
import json
import os
import subprocess
import sys

tag, wl = sys.argv[1], sys.argv[2]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
go = os.path.join(root, "gpurun_out")
pr = os.path.join(root, "profiles")

# launch list
rows = list(csv.reader(open(os.path.join(go, f"launches_{tag}.csv"))))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(lambda: [0, 0.0])
for x in data:
    if x["Metric Name"] != "gpu__time_duration.sum":
        continue
    k = x["Kernel Name"].split("(")[0]
    agg[k][0] += 1
    agg[k][1] += float(x["Metric Value"].replace(",", "")) / 1e3
tot = sum(v[1] for v in agg.values())
out = [f"ncu --metrics gpu__time_duration.sum --clock-control none -c 6000; python bench.py --steps 1 --warmup 3 "
       f"--no-baseline ({wl})", "per-launch times are cold-cache and serialised: compare shares, not absolutes"]
for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    out.append(f"{k[:60]:60s} launches={n:6d} total_us={us:11.1f} avg_us={us / n:9.2f} share={100 * us / tot:5.1f}%")
open(os.path.join(pr, f"launches_{tag}_{wl}.txt"), "w").write("\n".join(out) + "\n")

# full capture
raw = subprocess.run(["ncu", "-i", os.path.join(go, f"full_{tag}.ncu-rep"), "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(raw))
hdr, units = rows[0], rows[1]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct"]
txt = [f"ncu --set full --clock-control none --import-source on -s 40 -c 1 (gpu_round.sh {tag}, {wl})"]
traffic = {}
for r in rows[2:]:
    d = dict(zip(hdr, r))
    txt.append(d["Kernel Name"][:80])
    for k in keys:
        if k in d:
            txt.append(f"  {k} = {d[k]} {units[hdr.index(k)]}")
    st = [(k, d[k]) for k in hdr if k.startswith("smsp__average_warps_issue_stalled_") and
          k.endswith("_per_issue_active.ratio")]
    st = sorted(st, key=lambda kv: -float(kv[1] or 0))[:8]
    txt.append("  top stall reasons (warps per issue-active cycle): " +
               ", ".join(f"{k.split('stalled_')[1].split('_per')[0]}={float(v):.2f}" for k, v in st))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    b = sum(float(d[k].replace(",", "")) * scale.get(units[hdr.index(k)], 1)
            for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    name = "fused" if "k_fused" in d["Kernel Name"] else ("child_eval" if "k_child_eval" in d["Kernel Name"] else None)
    if name:
        traffic[name] = int(b)
open(os.path.join(pr, f"full_{tag}_{wl}.txt"), "w").write("\n".join(txt) + "\n")
tp = os.path.join(pr, "traffic_r01.json")
t = json.load(open(tp)) if os.path.exists(tp) else {}
t.update(traffic)
t["source"] = (f"dram__bytes_read.sum + dram__bytes_write.sum per launch from one ncu --set full capture "
               f"(profiles/full_{tag}_{wl}.txt)")
json.dump(t, open(tp, "w"), indent=1)
print("\n".join(out[:8]))
print("\n".join(txt))
