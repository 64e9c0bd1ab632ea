set -x
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?
timeout 300 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench rc=$?
tail -5 gpurun_out/smoke.log gpurun_out/gpu_tests.log gpurun_out/bench.log
