"""Summaries under profiles/ of round-2 captures: launch list shares and ncu
full-capture key metrics + stall reasons + the hottest SASS instructions.
Usage: python scripts/summarize_r02.py launches <csv> <out.txt> <title>
       python scripts/summarize_r02.py full <ncu-rep> <out.txt> <title>"""
import collections
import csv
import subprocess
import sys

mode, src, dst, title = sys.argv[1:5]
if mode == "launches":
    rows = list(csv.reader(open(src)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hd = rows[h]
    ki, vi = hd.index("Kernel Name"), hd.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[h + 1:]:
        if len(r) > vi:
            k = r[ki].split("(")[0]
            agg[k][0] += 1
            agg[k][1] += float(r[vi].replace(",", "")) / 1e3
    tot = sum(v[1] for v in agg.values())
    out = [title, "per-launch times are cold-cache and serialised: compare shares, not absolutes"]
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"{k[:70]:70s} launches={n:6d} total_us={us:11.1f} avg_us={us / n:9.2f} share={100 * us / tot:5.1f}%")
    open(dst, "w").write("\n".join(out) + "\n")
    print("\n".join(out[:8]))
    sys.exit(0)
raw = subprocess.run(["ncu", "-i", src, "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(raw))
hdr, units = rows[0], rows[1]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__sass_thread_inst_executed_op_dadd_pred_on.sum", "sm__sass_thread_inst_executed_op_dmul_pred_on.sum",
        "sm__sass_thread_inst_executed_op_dfma_pred_on.sum"]
txt = [title]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    txt.append(d["Kernel Name"][:100])
    for k in keys:
        if k in d:
            txt.append(f"  {k} = {d[k]} {units[hdr.index(k)]}")
    st = [(k, d[k]) for k in hdr if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
    tot = sum(float((v or "0").replace(",", "")) for _, v in st) or 1.0
    st = sorted(st, key=lambda kv: -float((kv[1] or "0").replace(",", "")))[:8]
    txt.append("  warp stall samples: " + ", ".join(
        f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')}={100 * float(v.replace(',', '')) / tot:.1f}%"
        for k, v in st))
sass = subprocess.run(["ncu", "-i", src, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                      text=True).stdout.splitlines()
srows = list(csv.reader(sass))
hs = [i for i, r in enumerate(srows) if r and r[0] == "Address"]
for j, start in enumerate(hs):
    end = hs[j + 1] - 1 if j + 1 < len(hs) else len(srows)
    h = srows[start]
    data = [r for r in srows[start + 1:end] if len(r) == len(h) and r[0].startswith("0x")]
    si, so = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
    tot = sum(float(r[si] or 0) for r in data) or 1.0
    top = sorted(range(len(data)), key=lambda i: -float(data[i][si] or 0))[:12]
    txt.append(f"  hottest SASS of kernel {j} (share of stall samples, instruction index):")
    for i in top:
        txt.append(f"    {100 * float(data[i][si]) / tot:5.1f}%  #{i:5d}  {data[i][so].strip()[:90]}")
open(dst, "w").write("\n".join(txt) + "\n")
print("\n".join(txt[:40]))
