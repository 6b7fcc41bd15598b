set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dense_gpu.py -x -q -k "golden or device or lazy_matches" > gpurun_out/pytest_d.log 2>&1; echo pd=$?
tail -2 gpurun_out/pytest_d.log
timeout 900 python bench.py > gpurun_out/bench_c3.log 2>&1; echo bench=$?
cat gpurun_out/bench_c3.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 > gpurun_out/bench_torchrun1.log 2>&1; echo tr=$?
tail -3 gpurun_out/bench_torchrun1.log
