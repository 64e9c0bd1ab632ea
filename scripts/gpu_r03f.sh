# round 2: meet in the middle with 2^dl ~ sqrt(children per block)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r03f.log 2>&1 || { echo build failed; tail gpurun_out/build_r03f.log; exit 1; }
for MT in 1; do
  timeout 60 python scripts/trace_cfg.py 4 18 > gpurun_out/trace_r03f_f7d18_mt$MT.log 2>&1; echo "== rastrigin d=18 mtab=$MT rc=$?"; grep -E "chain phase|exits" gpurun_out/trace_r03f_f7d18_mt$MT.log | tail -3
done
IBNB_TRACE=1 timeout 60 python scripts/prof_solve.py --config 4 --fid 9 --d 18 --solves 2 > gpurun_out/trace_r03f_f9d18.log 2>&1; echo "== styblinski d=18 rc=$?"; grep -E "chain phase" gpurun_out/trace_r03f_f9d18.log | tail -2
timeout 400 python bench.py --steps 5 --warmup 3 --no-baseline > gpurun_out/bench_r03f.log 2>&1; echo bench rc=$?; python -c "
import json; d=json.loads(open('gpurun_out/bench_r03f.log').read().strip().split('\n')[-1]); print(d['value'], d['ms_per_step'], {k: (round(v['s'],3), v['status']) for k,v in d.get('time_to_enclose_all_ten_n10000').items()})"
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "chain or n10000 or d20 or 20" --timeout 300 > gpurun_out/tests_r03f.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/tests_r03f.log; grep -E "^FAILED|^E  " gpurun_out/tests_r03f.log | head
