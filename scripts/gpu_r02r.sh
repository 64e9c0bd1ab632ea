# round 2: k_insert with one-scan tile prefixes -- Ackley n = 10 bench, graph-path tests
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02r.log 2>&1 || { echo build failed; exit 1; }
timeout 600 python bench.py --config 1 --steps 5 --warmup 3 --no-baseline > gpurun_out/bench1_r02r.log 2>&1; echo bench1 rc=$?; python -c "
import json; d=json.loads(open('gpurun_out/bench1_r02r.log').read().strip().split('\n')[-1]); print(d['value'], d['ms_per_step'], d['kernel_ms'])"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "solve or config or branch or fused" --timeout 300 > gpurun_out/quick_r02r.log 2>&1; echo quick rc=$?; tail -2 gpurun_out/quick_r02r.log; grep -E "^E |FAILED" gpurun_out/quick_r02r.log | head
