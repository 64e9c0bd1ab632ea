# tests + bench + explore + ncu launch list (1 GPU).  Usage: bash scripts/gpu_perf.sh <tag> "<explore runs>"
# Internal timeouts sum to < 1500 s: call gpurun with --timeout >= 1800.
TAG=${1:-p}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 420 python -m pytest tests -x -q -m gpu --timeout 120 > gpurun_out/gpu_tests_${TAG}.log 2>&1; rc=$?; echo tests rc=$rc; tail -2 gpurun_out/gpu_tests_${TAG}.log
[ $rc -ne 0 ] && { grep -E "^E |FAILED|Error" gpurun_out/gpu_tests_${TAG}.log | head -20; exit 0; }
timeout 240 python bench.py --steps 5 --warmup 3 --no-baseline > gpurun_out/bench_${TAG}.log 2>&1; rc=$?; echo bench rc=$rc
[ $rc -ne 0 ] && { grep -E "^E |FAILED|Error" gpurun_out/gpu_tests_${TAG}.log | head -20; exit 0; }
if [ -n "$2" ]; then timeout 400 python scripts/explore.py --runs "$2" --max-iter 20000 > gpurun_out/explore_${TAG}.log 2>&1; echo explore rc=$?; cut -c1-400 gpurun_out/explore_${TAG}.log; fi
timeout 240 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
  python scripts/prof_solve.py --config 1 --solves 2 > gpurun_out/launches_${TAG}.log 2>&1; echo launches rc=$?
IBNB_TRACE=1 timeout 120 python scripts/prof_solve.py --config 1 --solves 3 > gpurun_out/trace_${TAG}.log 2>&1; echo trace rc=$?
