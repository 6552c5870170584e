#!/bin/bash
# One GPU call (1 GPU): default bench (our arm, e2e + cpu_baseline), reference arm, ncu launch
# list of one solve of the bench workload, the dominant kernel's DRAM traffic at the bench
# size, and one `ncu --set full` capture per hot kernel class.  Outputs -> gpurun_out/.
set -x
mkdir -p gpurun_out
T=${TAG:-r02}
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu_$T.txt
timeout 900 python bench.py > gpurun_out/bench_ours_$T.json 2> gpurun_out/bench_ours_$T.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$T.json 2> gpurun_out/bench_ref_$T.err; echo "ref rc=$?"
# launch list: one solve (the JSON of this run is not a bench value; only the per-launch list is used)
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$T.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_launch_$T.log 2>&1
echo "ncu list rc=$?"
timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active \
    --clock-control none -k regex:bt2_ws --csv --log-file gpurun_out/bt2_traffic_$T.csv python tools/prof_run.py --n 32768 > gpurun_out/ncu_traffic_$T.log 2>&1
echo "ncu traffic rc=$?"
if [ "${FULL:-1}" = "1" ]; then
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:bt2_ws_kernel -c 1 -o gpurun_out/full_bt2_$T -f python tools/bt2_time.py 16384 9472 > gpurun_out/ncu_full_bt2_$T.log 2>&1; echo "full bt2 rc=$?"
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:tma_gemm_kernel --launch-skip 10 -c 1 -o gpurun_out/full_r2k_$T -f python tools/f2b_time.py 16384 > gpurun_out/ncu_full_r2k_$T.log 2>&1; echo "full r2k rc=$?"
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:symm_tma_kernel --launch-skip 10 -c 1 -o gpurun_out/full_symm_$T -f python tools/f2b_time.py 16384 > gpurun_out/ncu_full_symm_$T.log 2>&1; echo "full symm rc=$?"
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:panel_cqr_kernel --launch-skip 10 -c 1 -o gpurun_out/full_panel_$T -f python tools/f2b_time.py 16384 > gpurun_out/ncu_full_panel_$T.log 2>&1; echo "full panel rc=$?"
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:tma_gemm_kernel --launch-skip 262 -c 2 -o gpurun_out/full_bt1_$T -f python tools/prof_run.py --n 16384 > gpurun_out/ncu_full_bt1_$T.log 2>&1; echo "full bt1 rc=$?"
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:os_skew_mv_kernel --launch-skip 100 -c 1 -o gpurun_out/full_osmv_$T -f python tools/onestep_time.py 8192 > gpurun_out/ncu_full_osmv_$T.log 2>&1; echo "full osmv rc=$?"
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:chase_kernel -c 1 -o gpurun_out/full_chase_$T -f python tools/prof_run.py --n 16384 > gpurun_out/ncu_full_chase_$T.log 2>&1; echo "full chase rc=$?"
fi
