#!/bin/bash
# Copy one evidence pass (scripts/gpu_evidence.sh output in gpurun_out/) into profiles/$1.
R=${1:?round dir, e.g. r01}
D=profiles/$R
mkdir -p $D
cp gpurun_out/gpu.txt $D/gpu.txt
tail -1 gpurun_out/bench.log > $D/bench_lubm100.jsonl
tail -1 gpurun_out/bench_ref.log > $D/bench_reference_lubm100.jsonl
tail -1 gpurun_out/bench_u10000.log > $D/bench_lubm10k.jsonl
cp gpurun_out/launches_bench.csv $D/ncu_launches_bench_lubm100.csv
python scripts/ncu_summary.py $D/ncu_launches_bench_lubm100.csv > $D/ncu_launches_bench_lubm100_summary.txt
cp gpurun_out/qlaunches_u10000.csv $D/ncu_launches_queries_lubm10k.csv
python scripts/ncu_summary.py $D/ncu_launches_queries_lubm10k.csv > $D/ncu_launches_queries_lubm10k_summary.txt
cp gpurun_out/qprof_u10000.log $D/queries_lubm10k.txt
for K in k_bitmap_compact k_group_filter_rows; do
  if [ -f gpurun_out/prof_$K.ncu-rep ]; then
    ncu -i gpurun_out/prof_$K.ncu-rep --page raw --csv > $D/ncu_full_${K}_lubm100.csv 2>/dev/null
    python scripts/ncu_summary.py gpurun_out/prof_$K.ncu-rep > $D/ncu_full_${K}_lubm100_summary.txt
    python scripts/ncu_source.py gpurun_out/prof_$K.ncu-rep 25 > $D/ncu_source_${K}_lubm100.txt
  fi
done
python scripts/make_traffic.py $D/ncu_launches_bench_lubm100.csv profiles/ncu_traffic.json > /dev/null
python scripts/make_traffic.py $D/ncu_launches_queries_lubm10k.csv profiles/ncu_traffic_u10000.json > /dev/null
for P in prof_u10000_filter prof_u10000_expand; do
  if [ -f gpurun_out/$P.ncu-rep ]; then
    ncu -i gpurun_out/$P.ncu-rep --page raw --csv > $D/ncu_full_${P#prof_}.csv 2>/dev/null
    python scripts/ncu_summary.py gpurun_out/$P.ncu-rep > $D/ncu_full_${P#prof_}_summary.txt
    python scripts/ncu_source.py gpurun_out/$P.ncu-rep 25 > $D/ncu_source_${P#prof_}.txt
  fi
done
