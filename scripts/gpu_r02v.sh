# round 2: k_chain one-barrier phase 2 + register rank; sparse insertion + 1024-entry single-block list phase; full GPU tests, traces, benches
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02v.log 2>&1 || { echo build failed; tail gpurun_out/build_r02v.log; exit 1; }
for D in 16 18; do
  timeout 120 python scripts/trace_cfg.py 4 $D > gpurun_out/trace_r02v_f7d$D.log 2>&1; echo "== rastrigin d=$D rc=$?"; grep -E "chain phases|exits" gpurun_out/trace_r02v_f7d$D.log | tail -2; tail -1 gpurun_out/trace_r02v_f7d$D.log
done
timeout 120 python scripts/trace_cfg.py 1 > gpurun_out/trace_r02v_c1.log 2>&1; echo "== ackley n=10 rc=$?"; tail -7 gpurun_out/trace_r02v_c1.log
timeout 600 python bench.py --config 1 --steps 5 --warmup 3 --no-baseline > gpurun_out/bench1_r02v.log 2>&1; echo bench1 rc=$?; python -c "
import json; d=json.loads(open('gpurun_out/bench1_r02v.log').read().strip().split('\n')[-1]); print(d['value'], d['ms_per_step'], d['kernel_ms'])"
timeout 900 python bench.py --steps 5 --warmup 3 --no-baseline > gpurun_out/bench_r02v.log 2>&1; echo bench rc=$?; python -c "
import json; d=json.loads(open('gpurun_out/bench_r02v.log').read().strip().split('\n')[-1]); print(d['value'], d['ms_per_step'], d.get('time_to_enclose_all_ten_n10000'))"
bash scripts/gpu_tests.sh r02v
