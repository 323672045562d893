#!/bin/bash
# round-2 evidence: extra bench lines (LUBM-100, LUBM-10k), the N=2 path (two
# processes sharing the device), full-size power-law probe
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 600 python bench.py --workload lubm100 --steps 20 --warmup 5 > gpurun_out/bench_lubm100.log 2> gpurun_out/bench_lubm100.err; echo "lubm100 rc=$?"
timeout 1200 python bench.py --workload lubm10k --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_lubm10k.log 2> gpurun_out/bench_lubm10k.err; echo "lubm10k rc=$?"
timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --e2e-steps 1 > gpurun_out/bench_n2.log 2> gpurun_out/bench_n2.err; echo "n2 rc=$?"; tail -5 gpurun_out/bench_n2.err
timeout 1500 python scripts/probe_powerlaw.py --oracle > gpurun_out/probe_powerlaw.log 2>&1; echo "powerlaw rc=$?"; tail -30 gpurun_out/probe_powerlaw.log
for f in gpurun_out/bench_lubm100.log gpurun_out/bench_lubm10k.log gpurun_out/bench_n2.log; do echo "== $f"; head -c 1500 $f; echo; done
