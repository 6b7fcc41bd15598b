# round-1 call 4: faster CDF select + table exp; full GPU suite; benches; racecheck
set -x
timeout 1500 python -m pytest tests -m "gpu and not slow" -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 300 python bench.py --config c1 > gpurun_out/bench_c1.log 2>&1; echo c1=$?
timeout 300 python bench.py --config c2 > gpurun_out/bench_c2.log 2>&1; echo c2=$?
timeout 900 python bench.py > gpurun_out/bench_c3.log 2>&1; echo c3=$?
timeout 900 python bench.py --config c5 --steps 1 --warmup 1 > gpurun_out/bench_c5.log 2>&1; echo c5=$?
timeout 600 python scripts/sanitize_small.py > gpurun_out/plain_san.log 2>&1 && \
  timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard python scripts/sanitize_small.py > gpurun_out/racecheck.log 2>&1; echo race=$?
for f in gpurun_out/*.log; do echo "== $f"; tail -n 3 $f; done
