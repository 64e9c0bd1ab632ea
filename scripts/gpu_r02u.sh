# round 2: shared-word tests; potential children per chain iteration; k_chain full capture (d = 16) with the SASS source page
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02u.log 2>&1 || { echo build failed; tail gpurun_out/build_r02u.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "shared_incumbent" --timeout 300 > gpurun_out/shared_r02u.log 2>&1; echo shared rc=$?; tail -2 gpurun_out/shared_r02u.log
for D in 16 18; do
  timeout 120 python scripts/trace_cfg.py 4 $D > gpurun_out/trace_r02u_f7d$D.log 2>&1; echo "== rastrigin d=$D"; grep -E "chain phases|exits" gpurun_out/trace_r02u_f7d$D.log | tail -2
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_chain -s 1 -c 1 \
  -o gpurun_out/full_r02u_chain_d16 -f python scripts/prof_solve.py --config 4 --d 16 --solves 1 > gpurun_out/full_r02u.log 2>&1; echo full rc=$?
ncu -i gpurun_out/full_r02u_chain_d16.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_r02u_chain_d16.csv 2>/dev/null; echo sass rc=$?
ncu -i gpurun_out/full_r02u_chain_d16.ncu-rep --page raw --csv > gpurun_out/raw_r02u_chain_d16.csv 2>/dev/null
ls -la gpurun_out/ | tail -5
