set -x
mkdir -p gpurun_out
export RPLU_LAZY_BLOCK=16 PROFILE_STEPS=17
python scripts/profile_lazy.py > gpurun_out/prof_plain.log 2>&1; echo plain=$?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:lazy_pass4 --csv --log-file gpurun_out/pass4_q_launches.csv python scripts/profile_lazy.py > gpurun_out/ncu_launch.log 2>&1; echo l=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lazy_pass4 -s 7 -c 1 -f -o gpurun_out/pass4_q8 python scripts/profile_lazy.py > gpurun_out/ncu_q8.log 2>&1; echo q8=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lazy_pass4 -s 15 -c 1 -f -o gpurun_out/pass4_flush16 python scripts/profile_lazy.py > gpurun_out/ncu_flush.log 2>&1; echo fl=$?
