set -x
mkdir -p gpurun_out/final4
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final4/smoke.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/final4/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/final4/pytest_gpu.log
for c in c3f64 c3f32 c1 c2 c4 c4plan c5 gmres bary; do
  timeout 900 python bench.py --config $c > gpurun_out/final4/bench_$c.log 2>&1; echo $c=$?
done
timeout 900 python bench.py --impl reference > gpurun_out/final4/bench_ref.log 2>&1; echo ref=$?
for c in c3f64 c3f32 c1 c2 c4 c4plan c5 gmres bary ref; do tail -1 gpurun_out/final4/bench_$c.log | cut -c1-300; done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/final4/ncu_launches_bench.csv python bench.py --steps 1 --warmup 3 > gpurun_out/final4/ncu_bench.log 2>&1; echo ncu=$?
gzip -f gpurun_out/final4/ncu_launches_bench.csv
