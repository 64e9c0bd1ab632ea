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
a = ap.parse_args()
cfg = workloads.CONFIGS[a.config]
l, u = workloads.config_bounds(cfg)
ld = torch.tensor(l, device="cuda")
ud = torch.tensor(u, device="cuda")
o = pb.options(d=a.d or min(cfg["n"], 16), m=2, bmax=a.bmax or None)
ws = pb.Workspace(pb.solve_workspace_bytes(cfg["fid"], cfg["n"], o))
for _ in range(a.solves):
    r = pb.ib_solve_dev(cfg["fid"], ld, ud, cfg["eps"], cfg["eps"], o, workspace=ws)
torch.cuda.synchronize()
print(r.iters, r.evals, r.f_lo, r.f_hi, r.n_kernels)
