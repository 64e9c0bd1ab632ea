# round 2: two-phase k_insert (throughput regime) -- GPU tests, Ackley n = 10 bench, capture
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02o.log 2>&1 || { echo build failed; tail -5 gpurun_out/build_r02o.log; exit 1; }
timeout 600 python bench.py --config 1 --steps 5 --warmup 3 --no-baseline > gpurun_out/bench1_r02o.log 2>&1; echo bench1 rc=$?; python -c "
import json; d=json.loads(open('gpurun_out/bench1_r02o.log').read().strip().split('\n')[-1]); print(d['value'], d['ms_per_step'], d['kernel_ms'])"
bash scripts/gpu_tests.sh r02o
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_r02o_c1.csv \
  python bench.py --config 1 --steps 1 --warmup 3 --no-baseline > gpurun_out/launches_r02o_c1.log 2>&1; echo launches rc=$?
