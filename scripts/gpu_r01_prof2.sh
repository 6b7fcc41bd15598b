set -x
mkdir -p gpurun_out
python scripts/profile_gauss.py 400000 > gpurun_out/gauss_time.log 2>&1; cat gpurun_out/gauss_time.log
timeout 600 python bench.py --config c5 > gpurun_out/bench_c5.log 2>&1; echo c5=$?
cut -c1-700 gpurun_out/bench_c5.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mgs_arnoldi_kernel -c 1 -o gpurun_out/ncu_mgs python scripts/profile_consumers.py > gpurun_out/ncu_mgs.log 2>&1; echo ncu1=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bary_eval_kernel -c 1 -o gpurun_out/ncu_bary python scripts/profile_consumers.py > gpurun_out/ncu_bary.log 2>&1; echo ncu2=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gauss_gemv_kernel -c 1 -o gpurun_out/ncu_gauss_gemv17 python scripts/profile_gauss.py 200000 > gpurun_out/ncu_gauss.log 2>&1; echo ncu3=$?
