set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -m "gpu" -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -n 8 gpurun_out/pytest_gpu.log
