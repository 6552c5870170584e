#!/bin/bash
# GPU call: parity suite, GEMM tile sweep, bench (no CPU leg), ncu --set full of the F2B / BT1 GEMMs at n = 8192.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 ./tools/gemm_bench > gpurun_out/gemm_bench.txt 2>&1; echo "gemm_bench rc=$?"
timeout 900 python bench.py --no-cpu > gpurun_out/bench_v4.json 2> gpurun_out/bench_v4.err; echo "bench rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"symm_kernel|gemm_dmma_kernel" -s 40 -c 4 \
  -o gpurun_out/prof_f2b_gemm python tools/prof_run.py --n 8192 > gpurun_out/ncu_f2b.log 2>&1; echo "ncu f2b rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:gemm_dmma_kernel<64, 64, 16, 32, 32, 2, 1, 0, 0>" -s 60 -c 1 \
  -o gpurun_out/prof_bt1_z python tools/prof_run.py --n 8192 > gpurun_out/ncu_bt1.log 2>&1; echo "ncu bt1 rc=$?"
