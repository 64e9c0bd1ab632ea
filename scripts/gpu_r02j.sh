# round 2: grid k_chain with tree children, one-pass insertion kernel in the graph path, bench
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02j.log 2>&1 || { echo build failed; tail gpurun_out/build_r02j.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "chain_solve_parity or baseline_config or fused_graph" --timeout 300 > gpurun_out/quick_r02j.log 2>&1; echo quick rc=$?; tail -2 gpurun_out/quick_r02j.log; grep -E "^E " gpurun_out/quick_r02j.log | head -5
for f in 7 5; do timeout 120 python scripts/trace_fn.py $f 10000 2>&1 | grep -E "chain |^[a-z]+ 10000|rror" | tail -3; done
timeout 900 python scripts/chain_check.py 10000 > gpurun_out/chain_r02j.jsonl 2>&1; echo chain rc=$?
python -c "
import json
for l in open('gpurun_out/chain_r02j.jsonl'):
    try: r=json.loads(l)
    except Exception: print(l[:300]); continue
    print(r['fid'], r['n'], 'fused', r['fused']['s'], 'chain', r['chain']['s'], 'chainc', r['chainc']['s'], r['chain']['chain_launches'], 'same', r['same'])
"
timeout 600 python bench.py --config 1 --steps 5 --warmup 3 --no-baseline > gpurun_out/bench1_r02j.log 2>&1; echo bench1 rc=$?; python -c "
import json; d=json.loads(open('gpurun_out/bench1_r02j.log').read().strip().split('\n')[-1]); print(d['value'], d['ms_per_step'], d['kernel_ms'])"
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r02j.log 2>&1; echo bench rc=$?; cut -c1-600 gpurun_out/bench_r02j.log
bash scripts/gpu_tests.sh r02j
