# round 2: warp-voted children loops, HDR 56 (Levy d = 20) -- tests, d sweep, throughput-regime captures
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02n.log 2>&1 || { echo build failed; tail -5 gpurun_out/build_r02n.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "chain_solve_parity or d20 or sampled_children" --timeout 300 > gpurun_out/quick_r02n.log 2>&1; echo quick rc=$?; tail -2 gpurun_out/quick_r02n.log; grep -E "^E |FAILED" gpurun_out/quick_r02n.log | head -8
timeout 900 python scripts/dsweep.py 7,5,1 16,17,18,20 > gpurun_out/dsweep_r02n.jsonl 2>&1; echo dsweep rc=$?; python -c "
import json
for l in open('gpurun_out/dsweep_r02n.jsonl'):
    r=json.loads(l); print(r['fid'], r['d'], r['s'], r['iters'], round(r['box_evals_per_s']/1e9,1))"
for d in 16 18; do IBNB_TRACE=1 timeout 120 python scripts/trace_fn.py 7 10000 $d 2>&1 | grep -E "chain phases" | tail -1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_insert|k_list|k_child_eval' -s 30 -c 3 \
  -o gpurun_out/full_r02n_c1 -f python scripts/prof_solve.py --config 1 --solves 2 > gpurun_out/full_r02n_c1.log 2>&1; echo full rc=$?
