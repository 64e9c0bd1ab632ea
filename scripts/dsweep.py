"""Time to enclose vs the split width d (paper functions at n = 10,000 on their
domains, one warm-up + one timed solve each).  Usage: dsweep.py [fids] [ds] [n]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_01770_b200 as pb  # noqa: E402
import workloads  # noqa: E402

fids = [int(a) for a in sys.argv[1].split(",")] if len(sys.argv) > 1 else [7, 5, 1]
ds = [int(a) for a in sys.argv[2].split(",")] if len(sys.argv) > 2 else [16, 17, 18, 19, 20]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 10_000
for fid in fids:
    l, u = workloads.bounds(fid, n)
    ld, ud = torch.tensor(l, device="cuda"), torch.tensor(u, device="cuda")
    for d in ds:
        o = pb.options(d=d)
        ws = pb.Workspace(pb.solve_workspace_bytes(fid, n, o))
        pb.ib_solve_dev(fid, ld, ud, 1e-6, 1e-6, o, workspace=ws)
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = pb.ib_solve_dev(fid, ld, ud, 1e-6, 1e-6, o, workspace=ws)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        print(json.dumps({"fid": fid, "n": n, "d": d, "s": round(dt, 4), "iters": r.iters, "evals": r.evals,
                          "box_evals_per_s": r.evals / dt, "status": r.status, "enclosure": [r.f_lo, r.f_hi],
                          "chain_iters": r.prof["chain"]["units"]}), flush=True)
        del ws
