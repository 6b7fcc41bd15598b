# round-1 call 6: ncu captures of the select kernel, K5 and K7
set -x
for w in dense cauchy gauss; do
  timeout 600 python scripts/profile_kernels.py $w > gpurun_out/plain_$w.log 2>&1; echo plain_$w=$?
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense_select_kernel -s 2 -c 1 -o gpurun_out/prof_select python scripts/profile_kernels.py dense > gpurun_out/ncu_select.log 2>&1; echo n1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cauchy_mass_kernel -s 1 -c 1 -o gpurun_out/prof_k5 python scripts/profile_kernels.py cauchy > gpurun_out/ncu_k5.log 2>&1; echo n2=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gauss_gemv_kernel -s 1 -c 1 -o gpurun_out/prof_k7 python scripts/profile_kernels.py gauss > gpurun_out/ncu_k7.log 2>&1; echo n3=$?
for f in gpurun_out/*.log; do echo "== $f"; tail -n 2 $f; done
