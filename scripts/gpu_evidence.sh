#!/bin/bash
# Evidence pass (round profiles): bench line (configs[1]) + reference arm, ncu
# launch list of the same bench command (cold, serialised: compare shares), full
# captures of the dominant kernel classes, LUBM-10k bench line + query launch list.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
KR='k_(init|seed|guard|group|filter|zero|bitmap|seg|expand|prune|compact|enumerate|iota|gather|rank|scatter|push|and)|SortPairs|Onesweep'
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"$KR" --csv --log-file gpurun_out/launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_bench.log 2>&1
echo "launches rc=$?"
for K in k_bitmap_compact k_group_filter_rows; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 40 -c 4 \
    -o gpurun_out/prof_$K python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_full_$K.log 2>&1
  echo "full $K rc=$?"
done
timeout 1500 python bench.py --universities 10000 --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_u10000.log 2>&1; echo "bench u10000 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none \
  -k regex:"$KR" --csv --log-file gpurun_out/qlaunches_u10000.csv python scripts/prof_queries.py --universities 10000 --reps 2 > gpurun_out/qprof_u10000.log 2>&1
echo "qlaunches rc=$?"
python scripts/prof_queries.py --universities 10000 --reps 3 > gpurun_out/qprof_u10000.log 2>&1
# full captures at LUBM-10k: the push-form and pull-form edge evaluation of L7, the L1 expansion
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_push_edge|k_group_filter_rows' -c 3 \
  -o gpurun_out/prof_u10000_filter python scripts/prof_queries.py --universities 10000 --reps 1 --queries L7 > gpurun_out/ncu_full_u10000_filter.log 2>&1
echo "full u10000 filter rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_expand_lb -s 4 -c 2 \
  -o gpurun_out/prof_u10000_expand python scripts/prof_queries.py --universities 10000 --reps 1 --queries L1 > gpurun_out/ncu_full_u10000_expand.log 2>&1
echo "full u10000 expand rc=$?"
