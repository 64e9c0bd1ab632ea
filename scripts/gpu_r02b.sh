# round 2: GPU parity suite with k_chain, chain on/off comparison, bench
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02b.log 2>&1 || { echo build failed; tail gpurun_out/build_r02b.log; exit 1; }
bash scripts/gpu_tests.sh r02b
timeout 600 python scripts/chain_check.py 1000,10000 > gpurun_out/chain_r02b.jsonl 2>&1; echo chain rc=$?; cut -c1-600 gpurun_out/chain_r02b.jsonl
timeout 600 python bench.py > gpurun_out/bench_r02b.log 2>&1; echo bench rc=$?; cut -c1-1500 gpurun_out/bench_r02b.log
