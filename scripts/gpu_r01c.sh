# round-1 call 3: CUR + sharded parity, C5 bench, full-size ncu of the dense sweep
set -x
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 1200 python -m pytest tests -m "gpu and slow" -q > gpurun_out/pytest_slow.log 2>&1; echo slow=$?
timeout 900 python bench.py --config c5 --steps 1 --warmup 1 > gpurun_out/bench_c5.log 2>&1; echo c5=$?
CMD_F="python bench.py --steps 1 --warmup 1 --rank 8"
timeout 600 $CMD_F > gpurun_out/plain_f32k.log 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:dense_sweep_kernel -s 12 -c 1 -o gpurun_out/prof_dense_sweep_32k $CMD_F > gpurun_out/ncu_f32k.log 2>&1; echo ncuf=$?
for f in gpurun_out/*.log; do echo "== $f"; tail -n 3 $f; done
