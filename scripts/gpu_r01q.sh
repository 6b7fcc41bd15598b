set -x
timeout 900 python bench.py > gpurun_out/bench_c3.log 2>&1; echo c3=$?
for b in 4 5 6 8; do RPLU_LAZY_BLOCK=$b timeout 600 python bench.py --config c3f32 --steps 2 --warmup 1 > gpurun_out/bench_c3f32_b$b.log 2>&1; echo f$b=$?; done
CMD_L="python bench.py --steps 1 --warmup 2"
timeout 600 $CMD_L > gpurun_out/plain_l.log 2>&1 && \
  timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv $CMD_L > gpurun_out/ncu_l.log 2>&1; echo ncul=$?
for f in gpurun_out/*.log; do echo "== $f"; tail -n 2 $f | cut -c1-400; done
