#!/bin/bash
# One GPU call (1 GPU): default bench (our arm, e2e + cpu_baseline), reference arm, ncu launch
# list of one solve of the bench command, the dominant kernel's DRAM traffic at the bench size.
# Outputs -> gpurun_out/.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu.txt
timeout 900 python bench.py > gpurun_out/bench_ours.json 2> gpurun_out/bench_ours.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
# launch list: one solve (warm-up 0: the JSON of this run is not a bench value; only the per-launch list is used)
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
echo "ncu list rc=$?"
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active \
    --clock-control none -k regex:bt2_ws --csv --log-file gpurun_out/bt2_traffic.csv python tools/prof_run.py --n 32768 > gpurun_out/ncu_traffic.log 2>&1
echo "ncu traffic rc=$?"
