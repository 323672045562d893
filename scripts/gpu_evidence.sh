#!/bin/bash
# Evidence pass: bench line (configs[1]), ncu launch list of the same command
# (query kernels, cold/serialised: compare shares), one full capture of the top
# kernel, and the LUBM-10k scale line.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:'k_(init|seed|guard|group|filter|zero|bitmap|seg|expand|prune|compact|enumerate|iota|gather)|SortPairs' \
  --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_bench.log 2>&1
echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_group_filter -s 40 -c 8 \
  -o gpurun_out/prof_group_filter python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
timeout 1200 python bench.py --universities 10000 --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_u10000.log 2>&1; echo "bench u10000 rc=$?"
