set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_cauchy_gpu.py tests/test_cauchy_plan_gpu.py tests/test_distributed_gpu.py -x -q > gpurun_out/pytest_c.log 2>&1; echo pc=$?
tail -25 gpurun_out/pytest_c.log
timeout 600 python bench.py --config c2 > gpurun_out/bench_c2c.log 2>&1; echo b=$?
cut -c1-1200 gpurun_out/bench_c2c.log
