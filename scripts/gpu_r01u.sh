set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_distributed_gpu.py -x -q > gpurun_out/pytest_dist.log 2>&1; echo pdist=$?
timeout 900 python -m pytest tests/test_dense_gpu.py -x -q -k "sample or golden" > gpurun_out/pytest_dense_sample.log 2>&1; echo pds=$?
for f in gpurun_out/*.log; do echo "== $f"; tail -n 15 $f | cut -c1-300; done
