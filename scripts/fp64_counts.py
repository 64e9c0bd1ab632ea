"""Fold ncu counter CSVs (one per run of scripts/prof_solve.py) into executed
FP64-pipe instructions per unit of work for bench.py's roofline
(profiles/fp64_ops_r02.json).  Usage: fp64_counts.py out.json tag1.csv:tag1.log ..."""
import csv
import json
import sys
from collections import defaultdict

CLASS = {"k_chainc": "chain", "k_chain": "chain", "k_fused": "fused", "k_child_eval": "child_eval", "k_mono": "mono",
         "k_prep": "prep", "k_list": "list", "k_emit": "emit", "k_insert": "emit", "k_cand": "cand",
         "k_search": "search"}
FP = ("sm__sass_thread_inst_executed_op_dadd_pred_on.sum", "sm__sass_thread_inst_executed_op_dmul_pred_on.sum",
      "sm__sass_thread_inst_executed_op_dfma_pred_on.sum")


def kclass(name):
    base = name.split("(")[0].split("<")[0].replace("void ", "").strip().split("::")[-1]
    return CLASS.get(base)


out = {}
for arg in sys.argv[2:]:
    csvp, logp = arg.split(":")
    info = [json.loads(x) for x in open(logp) if x.startswith("{")][-1]
    rows = list(csv.reader(open(csvp)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hd = rows[h]
    ki, mi, vi, ii = hd.index("Kernel Name"), hd.index("Metric Name"), hd.index("Metric Value"), hd.index("ID")
    per = defaultdict(lambda: defaultdict(dict))
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        c = kclass(r[ki])
        if c:
            per[c][r[ii]][r[mi]] = float(r[vi].replace(",", ""))
    units = dict(info.get("units", {}))
    units.update({"chain": info["chain_iters"], "fused": info["fused_iters"], "child_eval": info["evals"]})
    res = {}
    for c, launches in per.items():
        fp = sum(m.get(k, 0.0) for m in launches.values() for k in FP)
        ns = sum(m.get("gpu__time_duration.sum", 0.0) for m in launches.values())
        issue = [m["smsp__issue_active.avg.pct_of_peak_sustained_active"] for m in launches.values()
                 if "smsp__issue_active.avg.pct_of_peak_sustained_active" in m]
        pipe = [m["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"] for m in launches.values()
                if "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active" in m]
        dram = sum(m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0) for m in launches.values())
        u = units.get(c)
        w = [m.get("gpu__time_duration.sum", 0.0) for m in launches.values()]
        wavg = lambda xs: sum(a * b for a, b in zip(xs, w)) / max(1e-9, sum(w)) if xs else None
        res[c] = {"launches": len(launches), "fp64_inst": fp, "units": u,
                  "unit": {"chain": "iteration", "fused": "iteration", "child_eval": "child box", "prep": "parent",
                           "mono": "candidate", "emit": "candidate", "cand": "child box"}.get(c),
                  "fp64_inst_per_unit": fp / u if u else None, "ncu_ms": ns / 1e6,
                  "issue_active_pct": wavg(issue), "fp64_pipe_pct": wavg(pipe),
                  "dram_bytes_per_launch": dram / max(1, len(launches))}
    out[str(info["fid"])] = {"n": info["n"], "iters": info["iters"], "kernels": res}
json.dump(out, open(sys.argv[1], "w"), indent=1)
print(json.dumps(out)[:2000])
