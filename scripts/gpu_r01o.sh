set -x
timeout 600 python scripts/profile_lazy.py > gpurun_out/plain_lazy.log 2>&1; echo p=$?
RPLU_LAZY_BLOCK=10 timeout 900 ncu --set full --clock-control none --import-source on -k regex:lazy_pass3_kernel -s 8 -c 1 -o gpurun_out/prof_lazy3 python scripts/profile_lazy.py > gpurun_out/ncu_lazy3.log 2>&1; echo n=$?
for b in 4 6 8; do RPLU_LAZY_RPT=8 RPLU_LAZY_BLOCK=$b timeout 600 python scripts/time_c3.py > gpurun_out/time_c3_r8b$b.log 2>&1; echo b$b=$?; done
timeout 900 python -m pytest tests/test_cauchy_plan_gpu.py tests/test_cauchy_gpu.py -q > gpurun_out/pytest_plan.log 2>&1; echo pp=$?
for f in gpurun_out/*.log; do echo "== $f"; tail -n 3 $f; done
