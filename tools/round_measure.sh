#!/bin/bash
# One GPU call (1 GPU): default bench (our arm), reference arm, ncu launch list of ONE timed
# step of the bench command (warm-up launches skipped with -s), the dominant kernel's DRAM
# traffic at the bench size, and one ncu --set full capture of it at n = 8192.
# Outputs -> gpurun_out/.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu.txt
timeout 900 python bench.py > gpurun_out/bench_ours.json 2> gpurun_out/bench_ours.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
L=$(python -c "import json;d=json.load(open('gpurun_out/bench_ours.json'));print(int(d['gpu_launches']//d['steps']))")
timeout 900 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain_launch.log 2>&1 && \
  timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none --csv -s $((3*L)) -c $((L+200)) \
    --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
echo "ncu list rc=$?"
timeout 300 python tools/prof_run.py --n 32768 > gpurun_out/plain_prof.log 2>&1 && \
  timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_op_dmma.sum \
    --clock-control none -k regex:bt2_ws --csv --log-file gpurun_out/bt2_traffic.csv python tools/prof_run.py --n 32768 > gpurun_out/ncu_traffic.log 2>&1
echo "ncu traffic rc=$?"
timeout 300 python tools/prof_run.py --n 8192 > gpurun_out/plain_prof8k.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:bt2_ws -c 1 -o gpurun_out/prof_bt2_full \
    python tools/prof_run.py --n 8192 > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
