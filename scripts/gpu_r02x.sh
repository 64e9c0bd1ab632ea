# round 2: k_chain one midpoint atomic per block again; sparse insertion warp test; A/B of the sparse insertion
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02x.log 2>&1 || { echo build failed; tail gpurun_out/build_r02x.log; exit 1; }
for D in 16 18; do
  timeout 120 python scripts/trace_cfg.py 4 $D > gpurun_out/trace_r02x_f7d$D.log 2>&1; echo "== rastrigin d=$D rc=$?"; grep -E "chain phases|exits" gpurun_out/trace_r02x_f7d$D.log | tail -2; tail -1 gpurun_out/trace_r02x_f7d$D.log
done
timeout 120 python scripts/trace_cfg.py 1 > gpurun_out/trace_r02x_c1.log 2>&1; echo "== ackley n=10 rc=$?"; grep -E "k_insert|t=.*iter=26" gpurun_out/trace_r02x_c1.log | tail -2
for SP in 1 0; do
IBNB_SPARSE=$SP timeout 600 python bench.py --config 1 --steps 5 --warmup 3 --no-baseline > gpurun_out/bench1_r02x_sp$SP.log 2>&1; echo bench1 sparse=$SP rc=$?; python -c "
import json; d=json.loads(open('gpurun_out/bench1_r02x_sp$SP.log').read().strip().split('\n')[-1]); print(d['value'], d['ms_per_step'], d['kernel_ms'])"
done
timeout 900 python bench.py --steps 5 --warmup 3 --no-baseline > gpurun_out/bench_r02x.log 2>&1; echo bench rc=$?; python -c "
import json; d=json.loads(open('gpurun_out/bench_r02x.log').read().strip().split('\n')[-1]); print(d['value'], d['ms_per_step'], {k: round(v['s'],3) for k,v in d.get('time_to_enclose_all_ten_n10000').items()})"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "solve or config or branch or fused or graph" --timeout 300 > gpurun_out/tests_r02x.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/tests_r02x.log; grep -E "^FAILED|^E  " gpurun_out/tests_r02x.log | head
