# round 2: ncu full capture (with source) of k_chain on Levy n = 10,000 d = 16 -- where its 20 us iterations go
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r03p.log 2>&1 || { echo build failed; exit 1; }
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_chain -s 1 -c 1 \
  -o gpurun_out/full_r03p_chain_levy -f python scripts/prof_solve.py --config 4 --fid 6 --d 16 --solves 1 > gpurun_out/full_r03p.log 2>&1; echo full rc=$?
ncu -i gpurun_out/full_r03p_chain_levy.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_r03p.csv 2>/dev/null; echo src rc=$?
