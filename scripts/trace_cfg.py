"""One traced solve of a BASELINE config (IBNB_TRACE=1): chunk log + fused phase times."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["IBNB_TRACE"] = "1"
import torch  # noqa: E402

import paper_2507_01770_b200 as pb  # noqa: E402
import workloads  # noqa: E402

cfg = workloads.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
d = int(sys.argv[2]) if len(sys.argv) > 2 else min(cfg["n"], 16)
l, u = workloads.config_bounds(cfg)
o = pb.options(d=d)
ws = pb.Workspace(pb.solve_workspace_bytes(cfg["fid"], cfg["n"], o))
ld, ud = torch.tensor(l, device="cuda"), torch.tensor(u, device="cuda")
for _ in range(2):
    r = pb.ib_solve_dev(cfg["fid"], ld, ud, cfg["eps"], cfg["eps"], o, workspace=ws)
print(r.status, r.iters, r.evals, r.f_lo, r.f_hi, r.n_surv, r.n_kernels)
