# explore runs (fid:n[:lo:hi[:m]] or config index), one GPU.  Usage: bash scripts/gpu_explore.sh <tag> "<runs>" [max_iter] [extra args]
TAG=${1:-x}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
for r in $(echo "$2" | tr ',' ' '); do
  timeout 300 python scripts/explore.py --runs "$r" --max-iter ${3:-100000} $4 >> gpurun_out/explore_${TAG}.log 2>&1 || echo "{\"run\": \"$r\", \"rc\": $?}" >> gpurun_out/explore_${TAG}.log
done
cut -c1-330 gpurun_out/explore_${TAG}.log
