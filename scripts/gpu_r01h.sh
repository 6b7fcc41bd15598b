# round-1 call 8: graph diagnostics for C1, K3 variants, sharded graph test
set -x
RPLU_DEBUG_GRAPH=1 timeout 300 python scripts/time_c1.py > gpurun_out/time_c1.log 2>&1; echo tc1=$?
timeout 600 python -m pytest tests/test_distributed_gpu.py -q > gpurun_out/pytest_dist.log 2>&1; echo pd=$?
for v in 0 1 2 3 4; do
  RPLU_SWEEP_VARIANT=$v timeout 600 python bench.py --steps 2 --warmup 1 > gpurun_out/bench_var$v.log 2>&1; echo var$v=$?
done
RPLU_DEBUG_GRAPH=1 timeout 300 python bench.py --config c1 > gpurun_out/bench_c1.log 2>&1; echo c1=$?
for f in gpurun_out/*.log; do echo "== $f"; tail -n 3 $f; done
