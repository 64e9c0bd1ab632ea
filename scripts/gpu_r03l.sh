# round 2 final evidence: GPU tests + smoke, bench lines (headline, Ackley n = 10), d sweep, FP64 counters, ncu full capture of k_chain (d = 18) and launch lists
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r03l.log 2>&1 || { echo build failed; exit 1; }
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r03l.log 2>&1; echo bench rc=$?; cut -c1-300 gpurun_out/bench_r03l.log | tail -1
timeout 400 python bench.py --config 1 --steps 10 --warmup 3 > gpurun_out/bench1_r03l.log 2>&1; echo bench1 rc=$?
timeout 600 python scripts/dsweep.py 7,3,1,6 16,17,18,20 > gpurun_out/dsweep_r03l.jsonl 2>&1; echo dsweep rc=$?
M=gpu__time_duration.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active
timeout 300 ncu --clock-control none -k regex:'k_chain|k_fused' --metrics $M --csv --log-file gpurun_out/cnt_r03l_f7d18.csv \
  python scripts/prof_solve.py --config 4 --fid 7 --d 18 --solves 1 > gpurun_out/cnt_r03l_f7d18.log 2>&1; echo counters d18 rc=$?
timeout 300 ncu --clock-control none -k regex:'k_child|k_prep|k_list|k_insert' --metrics $M --csv --log-file gpurun_out/cnt_r03l_c1.csv \
  python scripts/prof_solve.py --config 1 --solves 1 > gpurun_out/cnt_r03l_c1.log 2>&1; echo counters c1 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_chain -s 1 -c 1 \
  -o gpurun_out/full_r03l_chain_d18 -f python scripts/prof_solve.py --config 4 --d 18 --solves 1 > gpurun_out/full_r03l.log 2>&1; echo full rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_r03l.csv \
  python bench.py --steps 1 --warmup 3 --no-baseline --no-all-functions --no-secondary > gpurun_out/launches_r03l.log 2>&1; echo launches rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_r03l_c1.csv \
  python bench.py --config 1 --steps 1 --warmup 3 --no-baseline --no-all-functions --no-secondary > gpurun_out/launches_r03l_c1.log 2>&1; echo launches c1 rc=$?
bash scripts/gpu_tests.sh r03l
