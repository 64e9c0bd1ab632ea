# ncu --set full captures of the hot kernels (mid-solve launches) + FP64 counters.  Usage: bash scripts/gpu_full.sh <tag> [config]
TAG=${1:-f}
CFG=${2:-1}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
for K in k_list; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 8 -c 1 \
    -o gpurun_out/full_${K}_${TAG} -f python scripts/prof_solve.py --config $CFG --solves 1 > gpurun_out/full_${K}_${TAG}.log 2>&1; echo $K rc=$?
done
timeout 900 ncu --clock-control none -k regex:'k_child|k_prep|k_list|k_cand|k_mono|k_emit' \
  --metrics gpu__time_duration.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,sm__throughput.avg.pct_of_peak_sustained_elapsed \
  --csv --log-file gpurun_out/counters_${TAG}.csv python scripts/prof_solve.py --config $CFG --solves 1 > gpurun_out/counters_${TAG}.log 2>&1; echo counters rc=$?
