set -x
mkdir -p gpurun_out
timeout 600 python scripts/time_c1.py > gpurun_out/time_c1.log 2>&1; echo tc1=$?
cat gpurun_out/time_c1.log
RPLU_PERSIST_TRACE=1 timeout 600 python scripts/time_c1.py 2>&1 | sort | uniq -c | sort -rn | head -2
timeout 900 python -m pytest tests/test_dense_gpu.py -x -q -k "persistent or golden or c1" > gpurun_out/pytest_dense.log 2>&1; echo pd=$?
tail -3 gpurun_out/pytest_dense.log
