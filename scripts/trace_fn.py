"""One traced solve of a paper function at size n (IBNB_TRACE=1): fused phase times.  Usage: fid n [d]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["IBNB_TRACE"] = "1"
import torch  # noqa: E402

import paper_2507_01770_b200 as pb  # noqa: E402
import workloads  # noqa: E402

fid, n = int(sys.argv[1]), int(sys.argv[2])
d = int(sys.argv[3]) if len(sys.argv) > 3 else min(n, 16)
l, u = workloads.bounds(fid, n)
o = pb.options(d=d)
ws = pb.Workspace(pb.solve_workspace_bytes(fid, n, o))
ld, ud = torch.tensor(l, device="cuda"), torch.tensor(u, device="cuda")
for _ in range(2):
    r = pb.ib_solve_dev(fid, ld, ud, 1e-6, 1e-6, o, workspace=ws)
print(workloads.NAMES[fid], n, r.status, r.iters, r.f_lo, r.f_hi)
