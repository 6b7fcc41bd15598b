set -x
mkdir -p gpurun_out
RPLU_FORCE_SHARDED=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29535 bench.py --gpus 1 > gpurun_out/bench_sharded1.log 2>&1; echo s=$?
tail -3 gpurun_out/bench_sharded1.log | cut -c1-1500
