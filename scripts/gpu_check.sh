set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
free -g | head -2; nproc
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 300 python bench.py --config c1 --steps 3 --warmup 3 > gpurun_out/bench_c1.log 2>&1; echo benchc1=$?
timeout 900 python bench.py > gpurun_out/bench_c3.log 2>&1; echo bench=$?
tail -3 gpurun_out/pytest_gpu.log gpurun_out/smoke.log gpurun_out/bench_c1.log gpurun_out/bench_c3.log
