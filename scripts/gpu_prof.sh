# ncu evidence for the hot path (1 GPU).  Usage: bash scripts/gpu_prof.sh <tag> [config]
set -x
TAG=${1:-r01}
CFG=${2:-1}
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
# launch list (cold-cache, serialised: compare shares)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
  python scripts/prof_solve.py --config $CFG --solves 2 > gpurun_out/launches_${TAG}.log 2>&1; echo launches rc=$?
# FP64 / memory counters of the hot kernels (second solve)
timeout 900 ncu --clock-control none -k regex:'k_child|k_prep|k_partition|k_pool_stats' \
  --metrics gpu__time_duration.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__inst_executed_pipe_fp64.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,sm__throughput.avg.pct_of_peak_sustained_elapsed \
  --csv --log-file gpurun_out/counters_${TAG}.csv python scripts/prof_solve.py --config $CFG --solves 1 > gpurun_out/counters_${TAG}.log 2>&1; echo counters rc=$?
# full set of the dominant kernel, a mid-solve launch
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_child_lb -s 8 -c 1 \
  -o gpurun_out/prof_child_lb_${TAG} -f python scripts/prof_solve.py --config $CFG --solves 1 > gpurun_out/full_${TAG}.log 2>&1; echo full rc=$?
ls -la gpurun_out
