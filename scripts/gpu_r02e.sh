# round 2: chain with the first-order test in phase 1 -- traces, chain on/off at n = 10,000, GPU tests
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02e.log 2>&1 || { echo build failed; tail gpurun_out/build_r02e.log; exit 1; }
for f in 5 7 9 10 1 2; do timeout 120 python scripts/trace_fn.py $f 10000 2>&1 | grep -E "chain |^[a-z]+ 10000" | tail -3; done
timeout 600 python scripts/chain_check.py 10000 > gpurun_out/chain_r02e.jsonl 2>&1; echo chain rc=$?
python -c "
import json
for l in open('gpurun_out/chain_r02e.jsonl'):
    try: r=json.loads(l)
    except Exception: print(l[:200]); continue
    print(r['fid'], r['n'], 'fused', r['fused']['s'], 'chain', r['chain']['s'], r['chain']['chain_launches'], 'same', r['same'])
"
bash scripts/gpu_tests.sh r02e
