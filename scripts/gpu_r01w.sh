set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_dense_gpu.py tests/test_distributed_gpu.py -x -q -k "lazy or shard or delayed" > gpurun_out/pytest_lazy.log 2>&1; echo plazy=$?
tail -5 gpurun_out/pytest_lazy.log
timeout 900 python scripts/sweep_lazy_block.py f64 6,7,8,9,10,12 > gpurun_out/sweep_f64.log 2>&1; echo s64=$?
cat gpurun_out/sweep_f64.log
timeout 900 python scripts/sweep_lazy_block.py f32 5,6,8 > gpurun_out/sweep_f32.log 2>&1; echo s32=$?
cat gpurun_out/sweep_f32.log
