# round 2: non-separable chain objectives test their potential candidates warp-cooperatively (child_mono_ok_warp)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r03t.log 2>&1 || { echo build failed; tail gpurun_out/build_r03t.log; exit 1; }
timeout 400 python bench.py --steps 3 --warmup 3 --no-baseline > gpurun_out/bench_r03t.log 2>&1; echo bench rc=$?; python -c "
import json; d=json.loads(open('gpurun_out/bench_r03t.log').read().strip().split('\n')[-1]); print(d['value'], d['ms_per_step'], {k: (round(v['s'],3), v['status']) for k,v in d.get('time_to_enclose_all_ten_n10000').items()})"
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "chain or n10000 or headline or config" --timeout 300 > gpurun_out/tests_r03t.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/tests_r03t.log; grep -E "^FAILED|^E  " gpurun_out/tests_r03t.log | head
