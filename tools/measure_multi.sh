#!/bin/bash
# multi-GPU call (gpurun --gpus 4): distributed parity tests, bench at N = 2 and 4 (torchrun, NCCL),
# then BASELINE configs[4] (n = 65536) eigenvalues-only and nev = n/2 at N = 4 (input regenerated
# on the device each step: no pristine copy).
set -x
mkdir -p gpurun_out
TAG=${TAG:-r02}
nvidia-smi --query-gpu=index,name,memory.total --format=csv > gpurun_out/multi_gpus_$TAG.txt
[ "${PYTEST_MULTI:-1}" = "1" ] && timeout 600 python -m pytest tests/test_gpu_multi.py -q > gpurun_out/pytest_multi_$TAG.log 2>&1; echo "pytest multi rc=$?"
for N in ${BENCH_NS-2 4}; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600+N)) \
    bench.py --gpus $N --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/bench_${TAG}_n$N.json 2> gpurun_out/bench_${TAG}_n$N.err; echo "bench N=$N rc=$?"
done
if [ "${CONFIG4:-1}" = "1" ]; then
  BENCH_N=65536 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29700 \
    bench.py --gpus 4 --eigvals --regen --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/bench_${TAG}_c4_eigvals.json 2> gpurun_out/bench_${TAG}_c4_eigvals.err; echo "c4 eigvals rc=$?"
  BENCH_N=65536 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29701 \
    bench.py --gpus 4 --regen --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/bench_${TAG}_c4_vectors.json 2> gpurun_out/bench_${TAG}_c4_vectors.err; echo "c4 vectors rc=$?"
fi
