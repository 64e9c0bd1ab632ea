# round 2: cluster chain (k_chainc) -- traces, fused / grid chain / cluster chain at n = 10,000, GPU tests
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02h.log 2>&1 || { echo build failed; tail gpurun_out/build_r02h.log; exit 1; }
for cs in 1 2; do for f in 7 5 10 1; do IBNB_CHAIN=$cs timeout 120 python scripts/trace_fn.py $f 10000 2>&1 | grep -E "chain |^[a-z]+ 10000|rror" | tail -3; done; done
timeout 900 python scripts/chain_check.py 10000 > gpurun_out/chain_r02h.jsonl 2>&1; echo chain rc=$?
python -c "
import json
for l in open('gpurun_out/chain_r02h.jsonl'):
    try: r=json.loads(l)
    except Exception: print(l[:300]); continue
    print(r['fid'], r['n'], 'fused', r['fused']['s'], 'chain', r['chain']['s'], 'chainc', r['chainc']['s'], r['chainc']['chain_launches'], 'same', r['same'])
"
bash scripts/gpu_tests.sh r02h
M=gpu__time_duration.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active
for f in 7 5; do
timeout 600 ncu --clock-control none -k regex:'k_chain|k_fused' --metrics $M --csv --log-file gpurun_out/cnt_r02h_f$f.csv \
  python scripts/prof_solve.py --config 4 --fid $f --solves 1 > gpurun_out/cnt_r02h_f$f.log 2>&1; echo counters $f rc=$?
done
timeout 600 ncu --clock-control none -k regex:'k_child|k_mono|k_prep|k_list|k_emit|k_cand' --metrics $M --csv --log-file gpurun_out/cnt_r02h_c1.csv \
  python scripts/prof_solve.py --config 1 --solves 1 > gpurun_out/cnt_r02h_c1.log 2>&1; echo counters c1 rc=$?
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r02h.log 2>&1; echo bench rc=$?; cut -c1-800 gpurun_out/bench_r02h.log
