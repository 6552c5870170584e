#!/bin/bash
# One GPU call: default bench (our arm), reference arm, ncu launch list of the bench
# command, and one ncu --set full capture of the dominant kernel.  Outputs -> gpurun_out/.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu.txt
timeout 900 python bench.py > gpurun_out/bench_ours.json 2> gpurun_out/bench_ours.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain_launch.log 2>&1 && \
  timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo "ncu list rc=$?"
timeout 300 python tools/prof_run.py --n 32768 > gpurun_out/plain_prof.log 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:bt2_ws -c 1 -o gpurun_out/prof_bt2_full \
    python tools/prof_run.py --n 32768 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
