# round-1 call 2: cauchy parity, cauchy bench, ncu on the dense path
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m "gpu and not slow" -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py --config c2 --steps 3 --warmup 3 > gpurun_out/bench_c2.log 2>&1; echo c2=$?
timeout 900 python bench.py --config c4 --steps 2 --warmup 1 > gpurun_out/bench_c4.log 2>&1; echo c4=$?
timeout 600 python bench.py --config c3f32 > gpurun_out/bench_c3f32.log 2>&1; echo c3f32=$?
CMD_L="python bench.py --steps 1 --warmup 3"
timeout 600 $CMD_L > gpurun_out/plain_l.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv $CMD_L > gpurun_out/ncu_l.log 2>&1; echo ncul=$?
CMD_F="python bench.py --n 16384 --rank 64 --steps 1 --warmup 1"
timeout 600 $CMD_F > gpurun_out/plain_f.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dense_sweep_kernel -s 70 -c 2 -o gpurun_out/prof_dense_sweep $CMD_F > gpurun_out/ncu_f.log 2>&1; echo nccf=$?
for f in gpurun_out/*.log; do echo "== $f"; tail -n 4 $f; done
