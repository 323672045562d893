#!/bin/bash
# quick loop: core parity subset + bench (LUBM-100) + query profile (LUBM-10k)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fig12 or tiny or skewed or lubm_queries or watdiv or powerlaw or batch" > gpurun_out/pt.log 2>&1; tail -2 gpurun_out/pt.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
python scripts/prof_queries.py --universities ${U:-10000} --reps 2 > gpurun_out/qprof.log 2>&1; cat gpurun_out/qprof.log
