set -x
mkdir -p gpurun_out
export PROFILE_STEPS=13 RPLU_LAZY_BLOCK=6
RPLU_LAZY_ROLL=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:lazy_pass4 --csv --log-file gpurun_out/roll_launches.csv python scripts/profile_lazy.py > /dev/null 2>&1; echo b=$?
unset PROFILE_STEPS RPLU_LAZY_BLOCK
timeout 900 python -m pytest tests/test_dense_gpu.py -x -q -k "lazy" > gpurun_out/pytest_lazy.log 2>&1; echo plazy=$?
tail -2 gpurun_out/pytest_lazy.log
RPLU_LAZY_ROLL=1 timeout 900 python scripts/sweep_lazy_block.py f64 4,6,8 > gpurun_out/sweep_roll.log 2>&1; cat gpurun_out/sweep_roll.log
RPLU_LAZY_ROLL=0 timeout 900 python scripts/sweep_lazy_block.py f64 6 > gpurun_out/sweep_sync.log 2>&1; cat gpurun_out/sweep_sync.log
