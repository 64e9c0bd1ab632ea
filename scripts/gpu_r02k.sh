# round 2: FP64 counters per unit for every paper function (k_chain / k_fused) and the throughput regime; full capture of k_chain; launch list of the bench command
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02k.log 2>&1 || { echo build failed; exit 1; }
M=gpu__time_duration.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active
ARGS=""
for f in 1 2 3 4 5 6 7 8 9 10; do
timeout 300 ncu --clock-control none -k regex:'k_chain|k_fused' --metrics $M --csv --log-file gpurun_out/cnt_r02k_f$f.csv \
  python scripts/prof_solve.py --config 4 --fid $f --solves 1 > gpurun_out/cnt_r02k_f$f.log 2>&1; echo counters $f rc=$?
ARGS="$ARGS gpurun_out/cnt_r02k_f$f.csv:gpurun_out/cnt_r02k_f$f.log"
done
timeout 300 ncu --clock-control none -k regex:'k_child|k_prep|k_list|k_insert' --metrics $M --csv --log-file gpurun_out/cnt_r02k_c1.csv \
  python scripts/prof_solve.py --config 1 --solves 1 > gpurun_out/cnt_r02k_c1.log 2>&1; echo counters c1 rc=$?
python scripts/fp64_counts.py gpurun_out/fp64_ops_r02k.json $ARGS > /dev/null; echo fold rc=$?
python scripts/fp64_counts.py gpurun_out/fp64_ops_r02k_c1.json gpurun_out/cnt_r02k_c1.csv:gpurun_out/cnt_r02k_c1.log > /dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_chain -s 1 -c 1 \
  -o gpurun_out/full_r02k_chain -f python scripts/prof_solve.py --config 4 --solves 1 > gpurun_out/full_r02k.log 2>&1; echo full rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_r02k.csv \
  python bench.py --steps 1 --warmup 3 --no-baseline --no-all-functions --no-secondary > gpurun_out/launches_r02k.log 2>&1; echo launches rc=$?
