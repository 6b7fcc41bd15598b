set -x
mkdir -p gpurun_out
python scripts/profile_gauss.py 400000 > gpurun_out/gauss_time.log 2>&1; cat gpurun_out/gauss_time.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gauss_gemv_kernel -c 1 -o gpurun_out/ncu_gauss_gemv python scripts/profile_gauss.py 200000 > gpurun_out/ncu_gauss.log 2>&1; echo ncu=$?
timeout 600 python bench.py --config gmres > gpurun_out/bench_gmres.log 2>&1; echo gmres=$?
timeout 600 python bench.py --config bary > gpurun_out/bench_bary.log 2>&1; echo bary=$?
cut -c1-1500 gpurun_out/bench_gmres.log gpurun_out/bench_bary.log
