# Round evidence on one GPU: tests, bench (with clocks + cpu_baseline), ncu launch list of the bench command,
# FP64/DRAM counters of the hot kernel over one solve, one --set full capture.  Usage: bash scripts/gpu_round.sh <tag> [config]
TAG=${1:-r}
CFG=${2:-4}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo smoke rc=$?
timeout 600 python -m pytest tests -x -q -m gpu --timeout 300 > gpurun_out/gpu_tests_${TAG}.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/gpu_tests_${TAG}.log
timeout 600 python bench.py --config $CFG > gpurun_out/bench_${TAG}.log 2>&1; echo bench rc=$?; cut -c1-300 gpurun_out/bench_${TAG}.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_${TAG}.csv \
  python bench.py --config $CFG --steps 1 --warmup 3 --no-baseline --no-all-functions > gpurun_out/launches_${TAG}.log 2>&1; echo launches rc=$?
timeout 900 ncu --clock-control none -k regex:'k_fused|k_child|k_prep|k_list|k_cand|k_mono|k_emit|k_search' \
  --metrics gpu__time_duration.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,sm__throughput.avg.pct_of_peak_sustained_elapsed \
  --csv --log-file gpurun_out/counters_${TAG}.csv python scripts/prof_solve.py --config $CFG --solves 1 > gpurun_out/counters_${TAG}.log 2>&1; echo counters rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_fused|k_child_eval' -s 40 -c 1 \
  -o gpurun_out/full_${TAG} -f python scripts/prof_solve.py --config $CFG --solves 1 > gpurun_out/full_${TAG}.log 2>&1; echo full rc=$?
