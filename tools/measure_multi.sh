#!/bin/bash
# multi-GPU call (gpurun --gpus 4): distributed parity tests, bench at N = 2 and 4 (torchrun, NCCL),
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_multi.py -q > gpurun_out/pytest_multi.log 2>&1; echo "pytest multi rc=$?"
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600+N)) \
    bench.py --gpus $N --no-cpu --no-e2e > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; echo "bench N=$N rc=$?"
done
