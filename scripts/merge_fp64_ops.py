"""Merge fp64_counts.py outputs into profiles/fp64_ops_r02.json.
Usage: merge_fp64_ops.py file[:key_suffix] ...   (suffix e.g. @d18: keys fid@d18)"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(ROOT, "profiles", "fp64_ops_r02.json")
out = json.load(open(P)) if os.path.exists(P) else {}
for arg in sys.argv[1:]:
    path, _, suf = arg.partition(":")
    for fid, v in json.load(open(path)).items():
        key = fid + suf
        ent = out.setdefault(key, {"kernels": {}})
        for c, k in v["kernels"].items():
            ent["kernels"][c] = dict(k, n=v["n"])
json.dump(out, open(P, "w"), indent=1)
print(sorted(out.keys()))
