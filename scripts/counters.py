"""Summarise an ncu --csv counters log per kernel (sum over launches)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
data = []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(lambda: collections.defaultdict(float))
cnt = collections.Counter()
for d in data:
    k = d["Kernel Name"].split("(")[0].replace("void ib::", "")[:48]
    m = d["Metric Name"]
    v = float(d["Metric Value"].replace(",", "") or 0)
    agg[k][m] += v
    if m == "gpu__time_duration.sum":
        cnt[k] += 1
short = {"gpu__time_duration.sum": "ns", "sm__sass_thread_inst_executed_op_dadd_pred_on.sum": "dadd",
         "sm__sass_thread_inst_executed_op_dmul_pred_on.sum": "dmul", "sm__sass_thread_inst_executed_op_dfma_pred_on.sum": "dfma",
         "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64%", "dram__bytes_read.sum": "rdB",
         "dram__bytes_write.sum": "wrB", "sm__warps_active.avg.pct_of_peak_sustained_active": "warps%",
         "launch__registers_per_thread": "regs", "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm%"}
for k, ms in sorted(agg.items(), key=lambda kv: -kv[1]["gpu__time_duration.sum"]):
    out = []
    for m, v in ms.items():
        if "pct" in m or "registers" in m:
            v /= cnt[k]
        out.append(f"{short.get(m, m)}={v:.4g}")
    print(f"{k:42s} n={cnt[k]:3d} " + " ".join(out))
