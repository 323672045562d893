#!/bin/bash
# iteration loop: parity subset, LUBM-100 bench, LUBM-10k per-query launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "${K:-fig12 or tiny or skewed or lubm_queries or watdiv or powerlaw or batch or graph}" > gpurun_out/pt.log 2>&1; tail -2 gpurun_out/pt.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; python scripts/show_bench.py gpurun_out/bench.log
U=${U:-10000}
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control ${NCU_CACHE:-all} \
  -k regex:'k_(init|seed|guard|group|filter|zero|bitmap|seg|expand|prune|compact|enumerate|iota|gather)' \
  --csv --log-file gpurun_out/qlaunches_u$U.csv python scripts/prof_queries.py --universities $U --reps 1 > gpurun_out/ncu_qprof_u$U.log 2>&1
python scripts/prof_queries.py --universities $U --reps 3 2>&1 | grep -v "^ "
python scripts/ncu_summary.py gpurun_out/qlaunches_u$U.csv
