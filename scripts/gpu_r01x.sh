set -x
mkdir -p gpurun_out
python scripts/profile_lazy.py > gpurun_out/prof_plain.log 2>&1; echo plain=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lazy_pass4 -s 1 -c 1 -f -o gpurun_out/pass4_q2 python scripts/profile_lazy.py > gpurun_out/ncu_q2.log 2>&1; echo q2=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lazy_pass4 -s 4 -c 1 -f -o gpurun_out/pass4_flush python scripts/profile_lazy.py > gpurun_out/ncu_flush.log 2>&1; echo fl=$?
tail -3 gpurun_out/ncu_q2.log gpurun_out/ncu_flush.log
