# round 2 evidence: counters at the bench's launch configurations, full capture of k_chain (d = 18), launch list of the bench command, the bench line, GPU tests
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02q.log 2>&1 || { echo build failed; exit 1; }
M=gpu__time_duration.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active
timeout 300 ncu --clock-control none -k regex:'k_chain|k_fused' --metrics $M --csv --log-file gpurun_out/cnt_r02q_f7d18.csv \
  python scripts/prof_solve.py --config 4 --fid 7 --d 18 --solves 1 > gpurun_out/cnt_r02q_f7d18.log 2>&1; echo counters d18 rc=$?
timeout 300 ncu --clock-control none -k regex:'k_child|k_prep|k_list|k_insert' --metrics $M --csv --log-file gpurun_out/cnt_r02q_c1.csv \
  python scripts/prof_solve.py --config 1 --solves 1 > gpurun_out/cnt_r02q_c1.log 2>&1; echo counters c1 rc=$?
python scripts/fp64_counts.py gpurun_out/fp64_ops_r02q_f7d18.json gpurun_out/cnt_r02q_f7d18.csv:gpurun_out/cnt_r02q_f7d18.log > /dev/null
python scripts/fp64_counts.py gpurun_out/fp64_ops_r02q_c1.json gpurun_out/cnt_r02q_c1.csv:gpurun_out/cnt_r02q_c1.log > /dev/null
python scripts/merge_fp64_ops.py gpurun_out/fp64_ops_r02q_f7d18.json:@d18 gpurun_out/fp64_ops_r02q_c1.json && cp profiles/fp64_ops_r02.json gpurun_out/fp64_ops_r02_merged.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_chain -s 1 -c 1 \
  -o gpurun_out/full_r02q_chain_d18 -f python scripts/prof_solve.py --config 4 --d 18 --solves 1 > gpurun_out/full_r02q.log 2>&1; echo full rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_insert|k_child_eval' -s 30 -c 2 \
  -o gpurun_out/full_r02q_c1 -f python scripts/prof_solve.py --config 1 --solves 2 > gpurun_out/full_r02q_c1.log 2>&1; echo full c1 rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_r02q.csv \
  python bench.py --steps 1 --warmup 3 --no-baseline --no-all-functions --no-secondary > gpurun_out/launches_r02q.log 2>&1; echo launches rc=$?
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r02q.log 2>&1; echo bench rc=$?; cut -c1-400 gpurun_out/bench_r02q.log
bash scripts/gpu_tests.sh r02q
