"""Chain kernel check on the GPU: every paper function solved with the fused
path (IBNB_CHAIN=0), the grid chain (1) and the cluster chain (2), results
and wall time side by side."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_01770_b200 as pb  # noqa: E402
import workloads  # noqa: E402

ns = [int(a) for a in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1000, 10000]
fids = [int(a) for a in sys.argv[2].split(",")] if len(sys.argv) > 2 else list(range(1, 11))
d = int(sys.argv[3]) if len(sys.argv) > 3 else 16
for n in ns:
    for fid in fids:
        l, u = workloads.bounds(fid, n)
        row = {"fid": fid, "n": n}
        for mode in ("0", "1", "2"):
            os.environ["IBNB_CHAIN"] = mode
            pb.ib_solve(fid, l, u, 1e-6, 1e-6, pb.options(d=d), surv_cap=4)  # warm-up
            t = time.perf_counter()
            r = pb.ib_solve(fid, l, u, 1e-6, 1e-6, pb.options(d=d, profile=0), surv_cap=4)
            dt = time.perf_counter() - t
            rp = pb.ib_solve(fid, l, u, 1e-6, 1e-6, pb.options(d=d, profile=1), surv_cap=4)
            row[{"0": "fused", "1": "chain", "2": "chainc"}[mode]] = {
                "s": round(dt, 4), "status": r.status, "iters": r.iters, "evals": r.evals,
                "f": [r.f_lo, r.f_hi], "n_surv": r.n_surv, "w": r.max_width,
                "chain_launches": rp.prof["chain"]["launches"], "chain_iters": rp.prof["chain"]["units"],
                "fused_iters": rp.prof["fused"]["units"], "n_kernels": r.n_kernels,
                "lo0": float(r.lo[0][0]) if r.n_surv else None}
        key = lambda r: (r["iters"], r["n_surv"], r["status"], r["lo0"])
        row["same"] = key(row["fused"]) == key(row["chain"]) == key(row["chainc"])
        print(json.dumps(row), flush=True)
