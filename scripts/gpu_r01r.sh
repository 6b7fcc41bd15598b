set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_distributed_gpu.py -x -q > gpurun_out/pytest_dist.log 2>&1; echo pdist=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo smoke=$?
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1"
RPLU_FORCE_SHARDED=1 timeout 900 $TR --master-port 29518 bench.py --steps 2 --warmup 1 > gpurun_out/bench_sharded1_lazy.log 2>&1; echo shl=$?
RPLU_SHARD_UPDATE=eager RPLU_FORCE_SHARDED=1 timeout 900 $TR --master-port 29519 bench.py --steps 2 --warmup 1 > gpurun_out/bench_sharded1_eager.log 2>&1; echo she=$?
timeout 600 python scripts/profile_lazy.py > gpurun_out/plain_prof.log 2>&1 && \
  timeout 1800 ncu --set full --clock-control none --import-source on -k regex:lazy_pass3 --launch-skip 1 --launch-count 4 \
     -o gpurun_out/ncu_lazy_pass3 python scripts/profile_lazy.py > gpurun_out/ncu_full.log 2>&1; echo ncuf=$?
for f in gpurun_out/*.log; do echo "== $f"; tail -n 3 $f | cut -c1-600; done
