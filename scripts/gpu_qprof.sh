#!/bin/bash
mkdir -p gpurun_out
U=${U:-1000}
python scripts/prof_queries.py --universities $U --reps 3 > gpurun_out/qprof_u$U.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:'k_(init|seed|guard|group|filter|zero|bitmap|seg|expand|prune|compact|enumerate|iota|gather)|SortPairs|Onesweep' \
  --csv --log-file gpurun_out/qlaunches_u$U.csv python scripts/prof_queries.py --universities $U --reps 1 > gpurun_out/ncu_qprof_u$U.log 2>&1
echo "qlaunches rc=$?"
