#!/bin/bash
# iteration loop: build, a parity subset ($K), then a bench line ($BENCH_ARGS)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
if [ -n "$K" ]; then
  timeout ${T:-1500} python -m pytest tests/ -m gpu -x -q --timeout ${PT:-600} -k "$K" > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
fi
if [ -n "$BENCH" ]; then
  timeout ${TB:-900} python bench.py $BENCH > gpurun_out/bench.log 2> gpurun_out/bench.err
  echo "bench rc=$?"; tail -c 3000 gpurun_out/bench.log; tail -20 gpurun_out/bench.err
fi
