# round 2: D_MAX = 20, meet-in-the-middle children in k_chain -- tests, d sweep, all ten at d = 20
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02m.log 2>&1 || { echo build failed; tail -5 gpurun_out/build_r02m.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "chain_solve_parity or d20 or sampled_children" --timeout 300 > gpurun_out/quick_r02m.log 2>&1; echo quick rc=$?; tail -2 gpurun_out/quick_r02m.log; grep -E "^E |FAILED" gpurun_out/quick_r02m.log | head -8
timeout 900 python scripts/dsweep.py 7,5,1,10 16,17,18,19,20 > gpurun_out/dsweep_r02m.jsonl 2>&1; echo dsweep rc=$?; cut -c1-200 gpurun_out/dsweep_r02m.jsonl
IBNB_TRACE=1 timeout 120 python scripts/trace_fn.py 7 10000 20 2>&1 | grep -E "chain |^[a-z]+ 10000|rror" | tail -3
timeout 900 python scripts/chain_check.py 10000 1,2,3,4,5,7,8,9,10 20 > gpurun_out/chain_r02m.jsonl 2>&1; echo chain rc=$?
python -c "
import json
for l in open('gpurun_out/chain_r02m.jsonl'):
    try: r=json.loads(l)
    except Exception: print(l[:300]); continue
    print(r['fid'], r['n'], 'fused', r['fused']['s'], 'chain', r['chain']['s'], 'chainc', r['chainc']['s'], r['chain']['chain_launches'], 'same', r['same'])
"
bash scripts/gpu_tests.sh r02m
