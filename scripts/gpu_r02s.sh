# round 2 re-entry: verify the restored tree on the GPU (tests, smoke, bench line incl. throughput config)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
bash scripts/gpu_tests.sh r02s
timeout 600 python bench.py --config 1 --steps 5 --warmup 3 --no-baseline > gpurun_out/bench1_r02s.log 2>&1; echo bench1 rc=$?; python -c "
import json; d=json.loads(open('gpurun_out/bench1_r02s.log').read().strip().split('\n')[-1]); print(d['value'], d['ms_per_step'], d['kernel_ms'])"
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r02s.log 2>&1; echo bench rc=$?; cut -c1-600 gpurun_out/bench_r02s.log
