# round 2: lazy midpoint accumulators in child_eval_dev (graph + fused paths); Ackley n = 10 bench, graph/fused parity, smoke
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r03n.log 2>&1 || { echo build failed; tail gpurun_out/build_r03n.log; exit 1; }
timeout 400 python bench.py --config 1 --steps 10 --warmup 3 --no-baseline > gpurun_out/bench1_r03n.log 2>&1; echo bench1 rc=$?; python -c "
import json; d=json.loads(open('gpurun_out/bench1_r03n.log').read().strip().split('\n')[-1]); print(d['value'], d['ms_per_step'], d['kernel_ms'])"
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "solve or config or branch or fused or graph or eval" --timeout 300 > gpurun_out/tests_r03n.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/tests_r03n.log; grep -E "^FAILED|^E  " gpurun_out/tests_r03n.log | head
