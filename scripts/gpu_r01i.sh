set -x
timeout 600 python scripts/time_c3.py > gpurun_out/time_c3_auto.log 2>&1; echo a=$?
RPLU_GRAPH=always timeout 600 python scripts/time_c3.py > gpurun_out/time_c3_graph.log 2>&1; echo g=$?
timeout 300 python bench.py --config c1 > gpurun_out/bench_c1.log 2>&1; echo c1=$?
timeout 300 python bench.py --config c2 > gpurun_out/bench_c2.log 2>&1; echo c2=$?
for f in gpurun_out/*.log; do echo "== $f"; tail -n 4 $f; done
