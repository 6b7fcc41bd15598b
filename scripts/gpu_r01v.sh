set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -m "gpu" -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -n 8 gpurun_out/pytest_gpu.log
timeout 600 python scripts/time_c1.py > gpurun_out/time_c1.log 2>&1; cat gpurun_out/time_c1.log
RPLU_PERSIST_TRACE=1 timeout 600 python scripts/time_c1.py 2>&1 | grep rplu | head -2
timeout 900 python scripts/sweep_lazy_block.py f64 6 > gpurun_out/sweep_f64d.log 2>&1; cat gpurun_out/sweep_f64d.log
