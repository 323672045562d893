#!/bin/bash
# larger-scale bench line + ncu launch list (product kernels only) + full captures of the top kernels
mkdir -p gpurun_out
U=${U:-1000}
timeout 900 python bench.py --universities $U --steps 5 --warmup 3 --e2e-steps 1 > gpurun_out/bench_u$U.log 2>&1; echo "bench u$U rc=$?"
if [ -n "$NCU" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:'k_|Onesweep|Histogram|RadixSort' -c 600 --csv \
  --log-file gpurun_out/launches_u$U.csv python bench.py --universities $U --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_bench_u$U.log 2>&1
echo "launches rc=$?"
for K in ${KERNELS:-k_group_filter k_expand_lb k_seed_scatter}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s ${SKIP:-10} -c 2 \
    -o gpurun_out/prof_u${U}_$K python bench.py --universities $U --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_u${U}_$K.log 2>&1
  echo "$K rc=$?"
done
fi
