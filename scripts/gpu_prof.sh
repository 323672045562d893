#!/bin/bash
# ncu evidence: launch list of a short bench + one full capture of the top kernels.
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_bench.log 2>&1
echo "launches rc=$?"
for K in ${KERNELS:-k_group_filter k_expand_pass}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s ${SKIP:-20} -c 3 \
    -o gpurun_out/prof_$K python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_$K.log 2>&1
  echo "$K rc=$?"
done
