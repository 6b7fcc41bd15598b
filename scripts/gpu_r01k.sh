set -x
timeout 600 python scripts/profile_lazy.py > gpurun_out/plain_lazy.log 2>&1; echo p=$?
RPLU_LAZY_BLOCK=10 timeout 900 ncu --set full --clock-control none --import-source on -k regex:lazy_pass_kernel -s 6 -c 1 -o gpurun_out/prof_lazy python scripts/profile_lazy.py > gpurun_out/ncu_lazy.log 2>&1; echo n=$?
for b in 4 5; do RPLU_LAZY_BLOCK=$b timeout 600 python scripts/time_c3.py > gpurun_out/time_c3_b$b.log 2>&1; echo b$b=$?; done
for f in gpurun_out/*.log; do echo "== $f"; tail -n 4 $f; done
