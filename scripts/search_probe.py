"""R9 search alone: value, rounds and time per function / n (GPU)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_01770_b200 as pb  # noqa: E402
import workloads  # noqa: E402

ns = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "100,1000,10000").split(",")]
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 32
for n in ns:
    for fid in range(1, 11):
        l, u = workloads.bounds(fid, n)
        ld, ud = torch.tensor(l, device="cuda"), torch.tensor(u, device="cuda")
        pb.ib_search(fid, ld, ud, rounds)
        torch.cuda.synchronize()
        t = time.time()
        x, f, r = pb.ib_search(fid, ld, ud, rounds)
        torch.cuda.synchronize()
        dt = time.time() - t
        xc = x.cpu()
        print(json.dumps({"fn": workloads.NAMES[fid], "n": n, "f": f, "rounds": r, "ms": round(dt * 1e3, 3),
                          "x_min": float(xc.min()), "x_max": float(xc.max())}), flush=True)
