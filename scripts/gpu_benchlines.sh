#!/bin/bash
# bench lines only (LUBM-100 + reference arm, LUBM-10k) + smoke
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
timeout 1500 python bench.py --universities 10000 --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_u10000.log 2>&1; echo "bench u10000 rc=$?"
python scripts/prof_queries.py --universities 10000 --reps 3 > gpurun_out/qprof_u10000.log 2>&1
python scripts/show_bench.py gpurun_out/bench.log gpurun_out/bench_u10000.log
