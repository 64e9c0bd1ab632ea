cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 > gpurun_out/gpu_tests_x.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/gpu_tests_x.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-baseline > gpurun_out/bench_x.log 2>&1; echo bench rc=$?
timeout 1200 python scripts/explore.py --runs "$1" --max-iter ${2:-3000} > gpurun_out/explore.log 2>&1; echo explore rc=$?
cat gpurun_out/explore.log | cut -c1-700
