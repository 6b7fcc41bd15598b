set -x
mkdir -p gpurun_out
timeout 600 python scripts/time_e2e.py > gpurun_out/time_e2e.log 2>&1; echo e2e=$?
head -8 gpurun_out/time_e2e.log
grep -E "Memcpy|aten::to |cudaHostAlloc|cudaMalloc|pin|empty" gpurun_out/time_e2e.log | head -20
