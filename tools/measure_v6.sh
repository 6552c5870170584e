#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 300 ./tools/gemm_bench > gpurun_out/gemm_bench_v6.txt 2>&1; echo "gemm_bench rc=$?"
SKEWEIG_REORTH_DBG=1 timeout 300 python tools/prof_run.py --n 32768 > gpurun_out/reorth_dbg.txt 2>&1; echo "dbg rc=$?"
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/bench_v6.json 2> gpurun_out/bench_v6.err; echo "bench rc=$?"
