# round 2: chain exit statistics, launch list of the bench command, k_chain counters + full capture
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02c.log 2>&1 || { echo build failed; tail gpurun_out/build_r02c.log; exit 1; }
for f in 5 7 9 10 1; do timeout 120 python scripts/trace_fn.py $f 10000 2>&1 | grep -E "chain launches|^[a-z]+ 10000" ; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_r02c.csv \
  python bench.py --steps 1 --warmup 3 --no-baseline --no-all-functions --no-secondary > gpurun_out/launches_r02c.log 2>&1; echo launches rc=$?
timeout 600 ncu --clock-control none -k regex:'k_chain' -c 20 \
  --metrics gpu__time_duration.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,sm__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active \
  --csv --log-file gpurun_out/counters_r02c.csv python scripts/prof_solve.py --config 4 --solves 1 > gpurun_out/counters_r02c.log 2>&1; echo counters rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_chain -s 5 -c 1 \
  -o gpurun_out/full_r02c -f python scripts/prof_solve.py --config 4 --solves 1 > gpurun_out/full_r02c.log 2>&1; echo full rc=$?
