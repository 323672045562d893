#!/bin/bash
# full GPU suite + LUBM-100 bench + LUBM-100 per-query launch list (warm caches)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -x -m gpu > gpurun_out/pt_full.log 2>&1; tail -3 gpurun_out/pt_full.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; python scripts/show_bench.py gpurun_out/bench.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none \
  --csv --log-file gpurun_out/q100.csv python scripts/prof_queries.py --universities 100 --reps 2 > /dev/null 2>&1
python scripts/ncu_launches.py gpurun_out/q100.csv | tail -${TAILN:-60}
