"""Time to enclose vs the chain kernel's grid size (IBNB_CHAIN_GRID), paper
functions at n = 10,000.  Usage: gridsweep.py [fids] [grids] [d]"""
import json
import os
import subprocess
import sys

fids = sys.argv[1] if len(sys.argv) > 1 else "7,5,1"
grids = [int(a) for a in sys.argv[2].split(",")] if len(sys.argv) > 2 else [148, 128, 96, 74, 64, 48, 32]
d = sys.argv[3] if len(sys.argv) > 3 else "16"
here = os.path.dirname(os.path.abspath(__file__))
for g in grids:
    env = dict(os.environ, IBNB_CHAIN_GRID=str(g))
    out = subprocess.run([sys.executable, os.path.join(here, "dsweep.py"), fids, d], env=env, capture_output=True,
                         text=True).stdout
    for line in out.splitlines():
        r = json.loads(line)
        r["grid"] = g
        print(json.dumps(r), flush=True)
