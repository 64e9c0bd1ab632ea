# round 2 first GPU call: tightened parity suite + measured FP64 peak
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a_gpu.txt
(cd scripts/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu && ./fp64_peak) > gpurun_out/r02a_fp64_peak.json 2>&1
bash scripts/gpu_tests.sh r02a
