set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_distributed_gpu.py -x -q > gpurun_out/pytest_dist.log 2>&1; echo pdist=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo smoke=$?
for f in gpurun_out/*.log; do echo "== $f"; tail -n 5 $f | cut -c1-400; done
