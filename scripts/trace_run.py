"""Solve one problem with IBNB_TRACE output (fid n lo hi m [bmax])."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["IBNB_TRACE"] = "1"
import torch  # noqa: E402

import paper_2507_01770_b200 as pb  # noqa: E402

fid, n, lo, hi, m = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3]), float(sys.argv[4]), int(sys.argv[5])
bmax = int(sys.argv[6]) if len(sys.argv) > 6 else 0
o = pb.options(m=m, bmax=bmax or None)
ws = pb.Workspace(pb.solve_workspace_bytes(fid, n, o))
l = torch.full((n,), lo, dtype=torch.float64, device="cuda")
u = torch.full((n,), hi, dtype=torch.float64, device="cuda")
r = pb.ib_solve_dev(fid, l, u, 1e-6, 1e-6, o, workspace=ws)
print(r.status, r.iters, r.evals, r.f_lo, r.f_hi, r.n_surv)
