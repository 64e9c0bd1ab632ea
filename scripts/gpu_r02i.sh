# round 2: k_chain with stamped records (no grid barrier in the loop) -- chain tests first, traces, all functions, GPU tests
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02i.log 2>&1 || { echo build failed; tail gpurun_out/build_r02i.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "chain_solve_parity" --timeout 300 > gpurun_out/chaintest_r02i.log 2>&1; echo chaintest rc=$?; tail -3 gpurun_out/chaintest_r02i.log; grep -E "^E " gpurun_out/chaintest_r02i.log | head -5
for f in 7 5 10 1; do timeout 120 python scripts/trace_fn.py $f 10000 2>&1 | grep -E "chain |^[a-z]+ 10000|rror" | tail -3; done
timeout 900 python scripts/chain_check.py 10000 > gpurun_out/chain_r02i.jsonl 2>&1; echo chain rc=$?
python -c "
import json
for l in open('gpurun_out/chain_r02i.jsonl'):
    try: r=json.loads(l)
    except Exception: print(l[:300]); continue
    print(r['fid'], r['n'], 'fused', r['fused']['s'], 'chain', r['chain']['s'], 'chainc', r['chainc']['s'], r['chain']['chain_launches'], 'same', r['same'])
"
bash scripts/gpu_tests.sh r02i
