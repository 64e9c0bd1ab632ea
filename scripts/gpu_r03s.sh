# round 2: Levy chain potential candidates: warp-cooperative first-order test
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r03s.log 2>&1 || { echo build failed; tail gpurun_out/build_r03s.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "test_chain_solve_parity and (6-27 or 6-32 or 6-26)" --timeout 300 > gpurun_out/levy_tests_r03s.log 2>&1; echo levy chain tests rc=$?; tail -2 gpurun_out/levy_tests_r03s.log; grep -E "^FAILED|^E  " gpurun_out/levy_tests_r03s.log | head -20
IBNB_TRACE=1 timeout 60 python scripts/prof_solve.py --config 4 --fid 6 --d 16 --solves 2 > gpurun_out/trace_r03s_f6.log 2>&1; echo "== levy d=16 rc=$?"; grep -E "chain phase|exits" gpurun_out/trace_r03s_f6.log | tail -3; tail -1 gpurun_out/trace_r03s_f6.log
timeout 400 python bench.py --steps 3 --warmup 3 --no-baseline > gpurun_out/bench_r03s.log 2>&1; echo bench rc=$?; python -c "
import json; d=json.loads(open('gpurun_out/bench_r03s.log').read().strip().split('\n')[-1]); print(d['value'], d['ms_per_step'], {k: (round(v['s'],3), v['status']) for k,v in d.get('time_to_enclose_all_ten_n10000').items()})"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "n10000 or chain or levy or Levy" --timeout 300 > gpurun_out/tests_r03s.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/tests_r03s.log; grep -E "^FAILED|^E  " gpurun_out/tests_r03s.log | head
