# GPU tests (optionally a -k filter) + smoke.  Usage: bash scripts/gpu_tests.sh <tag> [pytest -k expr]
TAG=${1:-t}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
if [ -n "$2" ]; then K=(-k "$2"); else K=(); fi
timeout 900 python -m pytest tests -q -m gpu --timeout 300 "${K[@]}" > gpurun_out/gpu_tests_${TAG}.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/gpu_tests_${TAG}.log
grep -E "^FAILED|^E  " gpurun_out/gpu_tests_${TAG}.log | head -40
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/smoke_${TAG}.log
