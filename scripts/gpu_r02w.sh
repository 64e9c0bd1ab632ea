# round 2: k_chain: candidates tested in parallel before the phase-2 barrier, header by a warp butterfly, MITM template
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02w.log 2>&1 || { echo build failed; tail gpurun_out/build_r02w.log; exit 1; }
for D in 16 18; do
  timeout 120 python scripts/trace_cfg.py 4 $D > gpurun_out/trace_r02w_f7d$D.log 2>&1; echo "== rastrigin d=$D rc=$?"; grep -E "chain phases|exits" gpurun_out/trace_r02w_f7d$D.log | tail -2; tail -1 gpurun_out/trace_r02w_f7d$D.log
done
timeout 900 python bench.py --steps 5 --warmup 3 --no-baseline > gpurun_out/bench_r02w.log 2>&1; echo bench rc=$?; python -c "
import json; d=json.loads(open('gpurun_out/bench_r02w.log').read().strip().split('\n')[-1]); print(d['value'], d['ms_per_step'], {k: round(v['s'],3) for k,v in d.get('time_to_enclose_all_ten_n10000').items()})"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "chain or n10000 or headline or config" --timeout 300 > gpurun_out/chain_tests_r02w.log 2>&1; echo chain tests rc=$?; tail -2 gpurun_out/chain_tests_r02w.log; grep -E "^FAILED|^E  " gpurun_out/chain_tests_r02w.log | head
