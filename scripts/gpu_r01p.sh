set -x
timeout 900 python -m pytest tests/test_dense_gpu.py -q > gpurun_out/pytest_dense.log 2>&1; echo pd=$?
for b in 4 6 8; do RPLU_LAZY_BLOCK=$b timeout 600 python scripts/time_c3.py > gpurun_out/time_c3_q$b.log 2>&1; echo b$b=$?; done
RPLU_LAZY_RPT=4 RPLU_LAZY_BLOCK=6 timeout 600 python scripts/time_c3.py > gpurun_out/time_c3_q6r4.log 2>&1; echo r4=$?
RPLU_LAZY_BLOCK=8 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_lazy.csv python scripts/profile_lazy.py > gpurun_out/ncu_l.log 2>&1; echo l=$?
for f in gpurun_out/*.log; do echo "== $f"; tail -n 3 $f; done
