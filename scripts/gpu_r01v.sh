set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -m "gpu" -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -n 5 gpurun_out/pytest_gpu.log
timeout 600 python scripts/time_c1.py > gpurun_out/time_c1.log 2>&1; cat gpurun_out/time_c1.log
timeout 900 python bench.py > gpurun_out/bench_c3.log 2>&1; echo bench=$?
timeout 600 python bench.py --config c1 > gpurun_out/bench_c1.log 2>&1; echo benchc1=$?
timeout 600 python bench.py --config c3f32 > gpurun_out/bench_c3f32.log 2>&1; echo benchf32=$?
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.log 2>&1; echo benchref=$?
