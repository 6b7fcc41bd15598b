# round-1 call 11: 2-D lazy pass kernel + select/pivcol latency fixes
set -x
timeout 900 python -m pytest tests/test_dense_gpu.py -q -x > gpurun_out/pytest_dense.log 2>&1; echo pd=$?
for b in 4 6 8 10 12; do RPLU_LAZY_BLOCK=$b timeout 600 python scripts/time_c3.py > gpurun_out/time_c3_b$b.log 2>&1; echo b$b=$?; done
timeout 900 python bench.py --config c3f32 > gpurun_out/bench_c3f32.log 2>&1; echo c3f32=$?
for f in gpurun_out/*.log; do echo "== $f"; tail -n 4 $f; done
