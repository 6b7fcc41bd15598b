set -x
mkdir -p gpurun_out
timeout 600 python scripts/time_e2e.py > gpurun_out/time_e2e.log 2>&1; echo e2e=$?
timeout 900 python bench.py > gpurun_out/bench_c3.log 2>&1; echo bench=$?
cat gpurun_out/bench_c3.log
timeout 600 python bench.py --config c1 > gpurun_out/bench_c1.log 2>&1; echo benchc1=$?
cat gpurun_out/bench_c1.log
