# round 2: cluster chain (k_chainc) -- traces, fused / grid chain / cluster chain at n = 10,000, GPU tests
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02g.log 2>&1 || { echo build failed; tail gpurun_out/build_r02g.log; exit 1; }
for cs in 16 8; do for f in 7 5 10 1; do IBNB_CHAIN_CS=$cs timeout 120 python scripts/trace_fn.py $f 10000 2>&1 | grep -E "chain |^[a-z]+ 10000|rror" | tail -3; done; done
timeout 900 python scripts/chain_check.py 10000 > gpurun_out/chain_r02g.jsonl 2>&1; echo chain rc=$?
python -c "
import json
for l in open('gpurun_out/chain_r02g.jsonl'):
    try: r=json.loads(l)
    except Exception: print(l[:300]); continue
    print(r['fid'], r['n'], 'fused', r['fused']['s'], 'chain', r['chain']['s'], 'chainc', r['chainc']['s'], r['chainc']['chain_launches'], 'same', r['same'])
"
bash scripts/gpu_tests.sh r02g
