# round-1 call 7: msg-merged sharded step + graph replay; select with lighter CDF build
set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench_c3.log 2>&1; echo c3=$?
timeout 300 python bench.py --config c1 > gpurun_out/bench_c1.log 2>&1; echo c1=$?
RPLU_FORCE_SHARDED=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --size 8192 --pivots 64 --steps 2 --warmup 1 > gpurun_out/bench_sharded1.log 2>&1; echo sh=$?
RPLU_FORCE_SHARDED=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29518 bench.py --steps 2 --warmup 1 > gpurun_out/bench_sharded1_c3.log 2>&1; echo shc3=$?
for f in gpurun_out/*.log; do echo "== $f"; tail -n 3 $f; done
