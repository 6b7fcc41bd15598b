set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 900 python bench.py > gpurun_out/bench_c3.log 2>&1; echo c3=$?
timeout 600 python bench.py --config c3f32 > gpurun_out/bench_c3f32.log 2>&1; echo f32=$?
timeout 600 python bench.py --config c1 > gpurun_out/bench_c1.log 2>&1; echo c1=$?
timeout 600 python bench.py --config c2 > gpurun_out/bench_c2.log 2>&1; echo c2=$?
timeout 900 python bench.py --config c4 > gpurun_out/bench_c4.log 2>&1; echo c4=$?
timeout 900 python bench.py --config c5 > gpurun_out/bench_c5.log 2>&1; echo c5=$?
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo ref=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/ncu_launches_bench.csv python bench.py --steps 1 --warmup 3 > gpurun_out/ncu_bench.log 2>&1; echo ncu=$?
gzip -f gpurun_out/ncu_launches_bench.csv
