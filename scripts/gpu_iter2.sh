#!/bin/bash
# iteration: parity subset, LUBM-100 bench, LUBM-10k per-query kernel times,
# launch list of chosen queries, LUBM-100 host timeline
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "${K:-fig12 or lspm or tiny or skewed or lubm_queries or watdiv or powerlaw or batch}" > gpurun_out/pt.log 2>&1; tail -2 gpurun_out/pt.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; python scripts/show_bench.py gpurun_out/bench.log
U=${U:-10000}
python scripts/prof_queries.py --universities $U --reps 3 2>&1 | grep -v "^ "
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none \
  -k regex:'k_(init|seed|guard|group|filter|zero|bitmap|seg|expand|prune|compact|enumerate|iota|gather|rank|scatter|push|and)' \
  --csv --log-file gpurun_out/qlaunches_u$U.csv python scripts/prof_queries.py --universities $U --reps 1 --queries ${QS:-L1,L7} > gpurun_out/ncu_qprof_u$U.log 2>&1
echo "ncu rc=$?"; python scripts/ncu_launches.py gpurun_out/qlaunches_u$U.csv | head -80
timeout 300 python scripts/trace_latency.py > gpurun_out/trace.log 2>&1; echo "trace rc=$?"
