"""Run K solves of a BASELINE config (for ncu captures; no timing printed)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_01770_b200 as pb  # noqa: E402
import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--solves", type=int, default=2)
ap.add_argument("--bmax", type=int, default=0)
ap.add_argument("--d", type=int, default=0)
ap.add_argument("--fid", type=int, default=-1, help="a paper function on its own domain at the config's n")
a = ap.parse_args()
cfg = dict(workloads.CONFIGS[a.config])
if a.fid >= 0:
    cfg.update(fid=a.fid, lo=workloads.PAPER_DOMAIN[a.fid][0], hi=workloads.PAPER_DOMAIN[a.fid][1])
l, u = workloads.config_bounds(cfg)
ld = torch.tensor(l, device="cuda")
ud = torch.tensor(u, device="cuda")
o = pb.options(d=a.d or min(cfg["n"], 16), m=2, bmax=a.bmax or None)
ws = pb.Workspace(pb.solve_workspace_bytes(cfg["fid"], cfg["n"], o))
for _ in range(a.solves):
    r = pb.ib_solve_dev(cfg["fid"], ld, ud, cfg["eps"], cfg["eps"], o, workspace=ws)
torch.cuda.synchronize()
import json  # noqa: E402

print(json.dumps({"config": a.config, "fid": cfg["fid"], "n": cfg["n"], "iters": r.iters, "evals": r.evals,
                  "enclosure": [r.f_lo, r.f_hi], "n_kernels": r.n_kernels,
                  "chain_iters": r.prof["chain"]["units"], "fused_iters": r.prof["fused"]["units"],
                  "units": {c: v["units"] for c, v in r.prof.items()}}))
