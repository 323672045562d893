#!/bin/bash
# round-end evidence: full GPU parity suite, smoke, then scripts/gpu_evidence.sh
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pt_full.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
bash scripts/gpu_evidence.sh
python scripts/show_bench.py gpurun_out/bench.log gpurun_out/bench_u10000.log
tail -1 gpurun_out/bench_ref.log | cut -c1-300
