# build -> GPU tests -> bench -> ncu counters of the hot kernels.  Usage: bash scripts/gpu_iter.sh <tag> [config]
TAG=${1:-it}
CFG=${2:-1}
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 > gpurun_out/gpu_tests_${TAG}.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/gpu_tests_${TAG}.log
timeout 600 python bench.py --steps 5 --warmup 3 --config $CFG > gpurun_out/bench_${TAG}.log 2>&1; echo bench rc=$?
cut -c1-600 gpurun_out/bench_${TAG}.log
timeout 900 ncu --clock-control none -k regex:'k_child|k_prep|k_partition|k_pool_stats|k_radix' \
  --metrics gpu__time_duration.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,sm__throughput.avg.pct_of_peak_sustained_elapsed \
  --csv --log-file gpurun_out/counters_${TAG}.csv python scripts/prof_solve.py --config $CFG --solves 1 > gpurun_out/counters_${TAG}.log 2>&1; echo counters rc=$?
