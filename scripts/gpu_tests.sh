#!/bin/bash
# GPU parity suite (+ optional -k filter in $K), log to gpurun_out/pytest_gpu.log
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout ${T:-1800} python -m pytest tests/ -m gpu -x -q ${K:+-k "$K"} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
