#!/bin/bash
mkdir -p gpurun_out
U=${U:-1000}
for V in 0 1 2 3; do
  GSMART_FILTER_VARIANT=$V python scripts/prof_queries.py --universities $U --reps 3 > gpurun_out/var${V}_u$U.log 2>&1
  GSMART_FILTER_VARIANT=$V timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:'k_group_filter' --csv --log-file gpurun_out/var${V}_u$U.csv python scripts/prof_queries.py --universities $U --reps 1 > /dev/null 2>&1
done
