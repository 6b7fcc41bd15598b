set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
timeout 900 python scripts/sweep_lazy_block.py f64 6,8 > gpurun_out/sweep_narrow.log 2>&1; echo s=$?
cat gpurun_out/sweep_narrow.log
RPLU_LAZY_WIDE=1 timeout 900 python scripts/sweep_lazy_block.py f64 6,8 > gpurun_out/sweep_wide.log 2>&1; echo s=$?
cat gpurun_out/sweep_wide.log
RPLU_LAZY_WIDE=1 timeout 600 python -m pytest tests/test_dense_gpu.py -x -q -k "lazy" > gpurun_out/pytest_wide.log 2>&1; echo pw=$?
tail -2 gpurun_out/pytest_wide.log
