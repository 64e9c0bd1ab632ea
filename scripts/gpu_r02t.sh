# round 2: shared-word fix tests; chain phase timers (Rastrigin d = 16/18, Griewank d = 16, grid sizes); Ackley n = 10 trace
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02t.log 2>&1 || { echo build failed; tail gpurun_out/build_r02t.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "shared_incumbent" --timeout 300 > gpurun_out/shared_r02t.log 2>&1; echo shared rc=$?; tail -2 gpurun_out/shared_r02t.log
for D in 16 18; do
  timeout 120 python scripts/trace_cfg.py 4 $D > gpurun_out/trace_r02t_f7d$D.log 2>&1; echo "== rastrigin d=$D"; grep -E "chain phases|exits" gpurun_out/trace_r02t_f7d$D.log | tail -2
done
for G in 64 100; do
  IBNB_CHAIN_GRID=$G timeout 120 python scripts/trace_cfg.py 4 18 > gpurun_out/trace_r02t_f7d18_g$G.log 2>&1; echo "== rastrigin d=18 grid $G"; grep -E "chain phases" gpurun_out/trace_r02t_f7d18_g$G.log | tail -1
done
timeout 120 python scripts/prof_solve.py --config 4 --fid 3 --d 16 --solves 1 > /dev/null 2>&1
IBNB_TRACE=1 timeout 120 python scripts/prof_solve.py --config 4 --fid 3 --d 16 --solves 2 > gpurun_out/trace_r02t_f3.log 2>&1; echo "== griewank d=16"; grep -E "chain phases" gpurun_out/trace_r02t_f3.log | tail -1
timeout 120 python scripts/trace_cfg.py 1 > gpurun_out/trace_r02t_c1.log 2>&1; echo "== ackley n=10"; tail -12 gpurun_out/trace_r02t_c1.log
