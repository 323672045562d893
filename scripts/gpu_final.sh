#!/bin/bash
# round-end evidence: the full GPU suite (incl. full-size LUBM-1000/10k sampled
# parity), smoke(), the headline bench line and the extra workload lines
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout ${T:-3000} python -m pytest tests/ -m gpu -q --timeout 1500 ${K:+-k "$K"} > gpurun_out/pytest_gpu_all.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
if [ -z "$NOBENCH" ]; then
timeout 900 python bench.py > gpurun_out/bench_default.log 2> gpurun_out/bench_default.err; echo "bench rc=$?"; head -c 1200 gpurun_out/bench_default.log; echo
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.log 2> gpurun_out/bench_reference.err; echo "ref rc=$?"; head -c 600 gpurun_out/bench_reference.log; echo
fi
