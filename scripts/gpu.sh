#!/bin/bash
# The one gpurun wrapper.  Run on the GPU box from the repo root:
#   gpurun --timeout S -- 'bash scripts/gpu.sh <step> [<step> ...]'
# Every step builds first (once) and writes its logs under gpurun_out/.
#   tests     GPU parity suite; K="-k filter", T=suite timeout (s), PT=per-test timeout
#   bench     bench.py $BENCH (default: the headline line), then the reference arm
#   extra     bench lines of the other workloads (LUBM-100, LUBM-10k), N=2, power-law probe
#   ingest    f4 measurement (scripts/probe_ingest.py $INGEST)
#   ab        A/B of execution switches (scripts/ab_batch.py, $AB = --variants "...")
#   prof      ncu launch list of one warm batch of workload $W (default watdiv100m) and,
#             with KRN=<kernel regex>, one `ncu --set full` capture (KQ: queries run alone)
#   smoke     __graft_entry__.smoke()
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
W=${W:-watdiv100m}
for step in "$@"; do
  case $step in
  tests)
    timeout ${T:-3000} python -m pytest tests/ -m gpu -q --timeout ${PT:-1500} ${K:+-k "$K"} > gpurun_out/pytest_gpu.log 2>&1
    echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log ;;
  smoke)
    timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
    echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log ;;
  bench)
    timeout ${TB:-900} python bench.py ${BENCH:-} > gpurun_out/bench_default.log 2> gpurun_out/bench_default.err
    echo "bench rc=$?"; head -c 1500 gpurun_out/bench_default.log; echo
    timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.log 2> gpurun_out/bench_reference.err
    echo "ref rc=$?"; head -c 800 gpurun_out/bench_reference.log; echo ;;
  extra)
    timeout 600 python bench.py --workload lubm100 --steps 20 --warmup 5 > gpurun_out/bench_lubm100.log 2> gpurun_out/bench_lubm100.err; echo "lubm100 rc=$?"
    timeout 1200 python bench.py --workload lubm10k --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_lubm10k.log 2> gpurun_out/bench_lubm10k.err; echo "lubm10k rc=$?"
    timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --e2e-steps 1 > gpurun_out/bench_n2.log 2> gpurun_out/bench_n2.err; echo "n2 rc=$?"
    timeout 1500 python scripts/probe_powerlaw.py --oracle > gpurun_out/probe_powerlaw.log 2>&1; echo "powerlaw rc=$?"; tail -15 gpurun_out/probe_powerlaw.log ;;
  ingest)
    timeout 900 python scripts/probe_ingest.py ${INGEST:-} > gpurun_out/probe_ingest.log 2>&1; echo "ingest rc=$?"; tail -6 gpurun_out/probe_ingest.log ;;
  ab)
    timeout 900 python scripts/ab_batch.py --workload $W ${AB:-} > gpurun_out/ab.log 2>&1; echo "ab rc=$?"; cat gpurun_out/ab.log ;;
  prof)
    timeout ${TL:-900} ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file gpurun_out/launches_$W.csv python scripts/prof_batch.py --workload $W ${SEQ:+--sequential} \
      > gpurun_out/prof_launch.log 2>&1
    echo "launch list rc=$?"; python scripts/ncu_summary.py gpurun_out/launches_$W.csv | head -30
    if [ -n "${KRN:-}" ]; then
      timeout ${TF:-900} ncu --set full --clock-control none --import-source on --profile-from-start off \
        -k regex:$KRN -c ${NC:-3} -o gpurun_out/full_${W}_$KRN python scripts/prof_batch.py --workload $W --sequential \
        ${KQ:+--queries $KQ} > gpurun_out/prof_full.log 2>&1
      echo "full rc=$?"; python scripts/ncu_summary.py gpurun_out/full_${W}_$KRN.ncu-rep | head -20
    fi ;;
  *) echo "unknown step $step"; exit 2 ;;
  esac
done
