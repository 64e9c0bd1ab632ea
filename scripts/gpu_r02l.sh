# round 2: latency floor microbenchmark; chain with busy blocks excluded from the children
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
(cd scripts/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o chain_floor chain_floor.cu && ./chain_floor) > gpurun_out/chain_floor_r02l.json 2>&1; cat gpurun_out/chain_floor_r02l.json
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02l.log 2>&1 || { echo build failed; exit 1; }
for f in 7 5 1; do timeout 120 python scripts/trace_fn.py $f 10000 2>&1 | grep -E "chain |^[a-z]+ 10000|rror" | tail -3; done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "chain_solve_parity or separable_split or full_size" --timeout 300 > gpurun_out/quick_r02l.log 2>&1; echo quick rc=$?; tail -2 gpurun_out/quick_r02l.log; grep -E "^E " gpurun_out/quick_r02l.log | head -5
timeout 900 python scripts/chain_check.py 10000 > gpurun_out/chain_r02l.jsonl 2>&1; echo chain rc=$?
python -c "
import json
for l in open('gpurun_out/chain_r02l.jsonl'):
    try: r=json.loads(l)
    except Exception: print(l[:300]); continue
    print(r['fid'], r['n'], 'fused', r['fused']['s'], 'chain', r['chain']['s'], 'chainc', r['chainc']['s'], r['chain']['chain_launches'], 'same', r['same'])
"
