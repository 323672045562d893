#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python bench.py --universities 10000 --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_u10000.log 2>&1; echo "bench u10000 rc=$?"
python scripts/prof_queries.py --universities 10000 --reps 2 > gpurun_out/qprof_u10000.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:'k_(init|seed|guard|group|filter|zero|bitmap|seg|expand|prune|compact|enumerate|iota|gather)|SortPairs' \
  --csv --log-file gpurun_out/qlaunches_u10000.csv python scripts/prof_queries.py --universities 10000 --reps 1 > gpurun_out/ncu_qprof_u10000.log 2>&1
echo "ncu rc=$?"
