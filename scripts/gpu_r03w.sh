# round 2 final: the default bench line on the final HEAD (headline + all ten + BASELINE configs + cpu baseline + e2e) and Ackley n = 10
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r03w.log 2>&1 || { echo build failed; exit 1; }
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r03w.log 2>&1; echo bench rc=$?; cut -c1-400 gpurun_out/bench_r03w.log | tail -1
timeout 400 python bench.py --config 1 --steps 10 --warmup 3 > gpurun_out/bench1_r03w.log 2>&1; echo bench1 rc=$?
