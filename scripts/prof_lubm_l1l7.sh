python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_l1l7.csv python scripts/prof_batch.py --workload lubm10k --sequential --queries L1,L7 > gpurun_out/prof_l1.log 2>&1
echo rc=$?
python - <<'PY'
import csv,collections
rows=list(csv.reader(open("gpurun_out/launches_l1l7.csv")))
hi=next(i for i,r in enumerate(rows) if "Kernel Name" in r); h=rows[hi]
ki,mi,vi,idi=h.index("Kernel Name"),h.index("Metric Name"),h.index("Metric Value"),h.index("ID")
per=collections.OrderedDict()
for r in rows[hi+1:]:
    per.setdefault((int(r[idi]),r[ki].split("(")[0][:40]),{})[r[mi]]=float(r[vi].replace(",",""))
for (i,k),m in per.items():
    print(f"{i:4d} {k:40s} us={m['gpu__time_duration.sum']/1e3:8.1f} MB={(m['dram__bytes_read.sum']+m['dram__bytes_write.sum'])/1e6:8.2f}")
PY
