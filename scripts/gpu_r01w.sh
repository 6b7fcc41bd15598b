set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_dense_gpu.py -x -q -k "lazy" > gpurun_out/pytest_lazy.log 2>&1; echo plazy=$?
tail -5 gpurun_out/pytest_lazy.log
timeout 900 python scripts/sweep_lazy_block.py f64 5,6,8,10,12,16 > gpurun_out/sweep_f64.log 2>&1; echo s64=$?
cat gpurun_out/sweep_f64.log
