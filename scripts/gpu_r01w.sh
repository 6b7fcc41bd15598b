set -x
mkdir -p gpurun_out
timeout 900 python scripts/sweep_lazy_block.py f64 6,8 > gpurun_out/sweep_ip.log 2>&1; echo s=$?
cat gpurun_out/sweep_ip.log
RPLU_FLUSH_OOP=1 timeout 900 python scripts/sweep_lazy_block.py f64 6,8,10 > gpurun_out/sweep_oop.log 2>&1; echo s=$?
cat gpurun_out/sweep_oop.log
RPLU_FLUSH_OOP=1 RPLU_LAZY_BLOCK=6 PROFILE_STEPS=13 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:lazy_pass4 --csv --log-file gpurun_out/oop_launches.csv python scripts/profile_lazy.py > /dev/null 2>&1; echo n=$?
