set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_cur_gpu.py tests/test_consumers_gpu.py tests/test_abi.py -q -x > gpurun_out/pytest_f4.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_f4.log
timeout 600 python bench.py --config c5 > gpurun_out/bench_c5.log 2>&1; echo c5=$?
timeout 600 python bench.py --config gmres > gpurun_out/bench_gmres.log 2>&1; echo gmres=$?
timeout 600 python bench.py --config bary > gpurun_out/bench_bary.log 2>&1; echo bary=$?
cut -c1-1500 gpurun_out/bench_c5.log gpurun_out/bench_gmres.log gpurun_out/bench_bary.log
