"""Per-launch rows of an ncu --csv launch list: id, kernel, us, DRAM MB (optionally filtered)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
pat = sys.argv[2] if len(sys.argv) > 2 else ""
start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[start]
ki, mi, vi, idi = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
d = {}
for r in rows[start + 1:]:
    d.setdefault((int(r[idi]), r[ki]), {})[r[mi]] = float(r[vi].replace(",", ""))
for (i, k), m in sorted(d.items()):
    if pat and pat not in k:
        continue
    t = m.get("gpu__time_duration.sum", 0) / 1000
    b = (m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)) / 1e6
    print(f"{i:4d} {k[:40]:40s} us={t:9.1f} MB={b:9.1f} GB/s={b / max(t, 1e-9) * 1e3:8.1f}")
