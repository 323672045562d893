#!/bin/bash
# ncu evidence for one workload ($W, default watdiv100m): the launch list of one
# warm query batch (device time + DRAM bytes per launch) and, if $KRN is set, one
# `--set full` capture of that kernel ($KQ: queries to run alone, e.g. C1).
mkdir -p gpurun_out
W=${W:-watdiv100m}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout ${TL:-900} ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/launches_$W.csv python scripts/prof_batch.py --workload $W ${SEQ:+--sequential} \
  > gpurun_out/prof_launch.log 2>&1
echo "launch list rc=$?"; tail -3 gpurun_out/prof_launch.log
python scripts/ncu_summary.py gpurun_out/launches_$W.csv | head -30
if [ -n "$KRN" ]; then
  timeout ${TF:-900} ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:$KRN -c ${NC:-3} -o gpurun_out/full_${W}_$KRN python scripts/prof_batch.py --workload $W --sequential \
    ${KQ:+--queries $KQ} > gpurun_out/prof_full.log 2>&1
  echo "full rc=$?"; tail -3 gpurun_out/prof_full.log
  python scripts/ncu_summary.py gpurun_out/full_${W}_$KRN.ncu-rep | head -20
fi
