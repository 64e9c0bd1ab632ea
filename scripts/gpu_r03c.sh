# round 2: listed candidates filtered by the warp's smallest midpoint value before the first-order test; traces, chain parity, bench
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r03c.log 2>&1 || { echo build failed; tail gpurun_out/build_r03c.log; exit 1; }
for D in 16 18; do
  timeout 60 python scripts/trace_cfg.py 4 $D > gpurun_out/trace_r03c_f7d$D.log 2>&1; echo "== rastrigin d=$D rc=$?"; grep -E "chain phase|exits" gpurun_out/trace_r03c_f7d$D.log | tail -3
done
for F in 6 3 9; do
IBNB_TRACE=1 timeout 60 python scripts/prof_solve.py --config 4 --fid $F --d 16 --solves 2 > gpurun_out/trace_r03c_f$F.log 2>&1; echo "== fid $F d=16 rc=$?"; grep -E "chain phase|exits" gpurun_out/trace_r03c_f$F.log | tail -3
done
timeout 400 python bench.py --steps 5 --warmup 3 --no-baseline > gpurun_out/bench_r03c.log 2>&1; echo bench rc=$?; python -c "
import json; d=json.loads(open('gpurun_out/bench_r03c.log').read().strip().split('\n')[-1]); print(d['value'], d['ms_per_step'], {k: (round(v['s'],3), v['status']) for k,v in d.get('time_to_enclose_all_ten_n10000').items()})"
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "chain or n10000 or headline or config" --timeout 300 > gpurun_out/tests_r03c.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/tests_r03c.log; grep -E "^FAILED|^E  " gpurun_out/tests_r03c.log | head
