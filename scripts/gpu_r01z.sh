set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_cauchy_gpu.py tests/test_cauchy_plan_gpu.py tests/test_distributed_gpu.py -x -q > gpurun_out/pytest_c.log 2>&1; echo pc=$?
tail -3 gpurun_out/pytest_c.log
timeout 600 python bench.py --config c2 > gpurun_out/bench_c2.log 2>&1; echo b=$?
cut -c1-400 gpurun_out/bench_c2.log
PROFILE_NOGRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2_launches.csv python scripts/profile_c2.py > /dev/null 2>&1; echo l=$?
