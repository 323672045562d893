#!/bin/bash
# round-end refresh: full GPU parity suite, smoke, bench lines (LUBM-100 + reference, LUBM-10k),
# ncu launch lists of the bench command and of the LUBM-10k queries
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pt_full.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
KR='k_(init|seed|guard|group|filter|zero|bitmap|seg|expand|prune|compact|enumerate|iota|gather|rank|scatter|push|and|phase2)|SortPairs|Onesweep'
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"$KR" --csv --log-file gpurun_out/launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_bench.log 2>&1
echo "launches rc=$?"
timeout 1500 python bench.py --universities 10000 --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_u10000.log 2>&1; echo "bench u10000 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none \
  -k regex:"$KR" --csv --log-file gpurun_out/qlaunches_u10000.csv python scripts/prof_queries.py --universities 10000 --reps 2 > /dev/null 2>&1
echo "qlaunches rc=$?"
python scripts/prof_queries.py --universities 10000 --reps 3 > gpurun_out/qprof_u10000.log 2>&1
python scripts/show_bench.py gpurun_out/bench.log gpurun_out/bench_u10000.log
tail -1 gpurun_out/bench_ref.log | cut -c1-300
