# round 2 final: d sweep on the final HEAD
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r03x.log 2>&1 || { echo build failed; exit 1; }
timeout 600 python scripts/dsweep.py 7,3,1,6 16,17,18,20 > gpurun_out/dsweep_r03x.jsonl 2>&1; echo dsweep rc=$?
