set -x
timeout 600 python scripts/profile_lazy.py > gpurun_out/plain_lazy.log 2>&1; echo p=$?
RPLU_LAZY_BLOCK=10 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_lazy.csv python scripts/profile_lazy.py > gpurun_out/ncu_l.log 2>&1; echo l=$?
RPLU_LAZY_BLOCK=10 timeout 900 ncu --set full --clock-control none --import-source on -k regex:lazy_pass2_kernel -s 6 -c 1 -o gpurun_out/prof_lazy2 python scripts/profile_lazy.py > gpurun_out/ncu_lazy2.log 2>&1; echo n=$?
for f in gpurun_out/*.log; do echo "== $f"; tail -n 2 $f; done
