"""Run BASELINE configs / paper functions with an iteration cap and report progress."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2507_01770_b200 as pb  # noqa: E402
import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--runs", default="2,3")  # config indices, or fid:n[:lo:hi]
ap.add_argument("--max-iter", type=int, default=2000)
ap.add_argument("--bmax", type=int, default=0)
ap.add_argument("--m", type=int, default=2)
ap.add_argument("--d", type=int, default=0)
ap.add_argument("--eps", type=float, default=1e-6)
ap.add_argument("--profile", type=int, default=1, help="1: per-kernel CUDA events (eager launches); 0: graph / fused path, timed")
ap.add_argument("--repeat", type=int, default=1)
a = ap.parse_args()
for spec in a.runs.split(","):
    m = a.m
    if ":" in spec:
        p = spec.split(":")
        fid, n = int(p[0]), int(p[1])
        if len(p) > 4:
            m = int(p[4])
        if len(p) > 2 and p[2] != "":
            l, u = np.full(n, float(p[2])), np.full(n, float(p[3]))
        else:
            l, u = workloads.bounds(fid, n)
        name = f"{workloads.NAMES[fid]}-n{n}"
    else:
        cfg = workloads.CONFIGS[int(spec)]
        fid, n = cfg["fid"], cfg["n"]
        l, u = workloads.config_bounds(cfg)
        name = cfg["name"]
    o = pb.options(d=a.d or min(n, 16), m=m, bmax=a.bmax or None, max_iter=a.max_iter, profile=a.profile)
    ws = pb.Workspace(pb.solve_workspace_bytes(fid, n, o))
    ld, ud = torch.tensor(l, device="cuda"), torch.tensor(u, device="cuda")
    try:
        for _ in range(a.repeat):  # the last repeat is timed (earlier ones warm up)
            torch.cuda.synchronize()
            t0 = time.time()
            r = pb.ib_solve_dev(fid, ld, ud, a.eps, a.eps, o, workspace=ws)
            torch.cuda.synchronize()
            dt = time.time() - t0
        print(json.dumps({"run": name, "m": m, "d": o.d, "status": r.status, "iters": r.iters, "evals": r.evals, "f_lo": r.f_lo,
                          "f_hi": r.f_hi, "f_search": r.f_search, "n_surv": r.n_surv, "peak_pool": r.peak_pool, "max_width": r.max_width,
                          "wall_s": dt, "kernel_ms": {k: round(v["ms"], 2) for k, v in r.prof.items()}}), flush=True)
    except Exception as e:
        print(json.dumps({"run": name, "error": str(e)[:300], "wall_s": time.time() - t0}), flush=True)
    del ws
    torch.cuda.empty_cache()
