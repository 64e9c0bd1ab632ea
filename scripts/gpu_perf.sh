# tests + bench + explore + ncu launch list of the bench config.  Usage: bash scripts/gpu_perf.sh <tag> "<explore runs>"
TAG=${1:-p}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 > gpurun_out/gpu_tests_${TAG}.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/gpu_tests_${TAG}.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-baseline > gpurun_out/bench_${TAG}.log 2>&1; echo bench rc=$?
if [ -n "$2" ]; then timeout 1200 python scripts/explore.py --runs "$2" --max-iter 20000 > gpurun_out/explore_${TAG}.log 2>&1; echo explore rc=$?; cut -c1-400 gpurun_out/explore_${TAG}.log; fi
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
  python scripts/prof_solve.py --config 1 --solves 2 > gpurun_out/launches_${TAG}.log 2>&1; echo launches rc=$?
IBNB_TRACE=1 timeout 300 python scripts/prof_solve.py --config 1 --solves 3 > gpurun_out/trace_${TAG}.log 2>&1; echo trace rc=$?
