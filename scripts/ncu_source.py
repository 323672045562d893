"""Top source lines by warp-stall samples from `ncu --page source --csv --print-source cuda`."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
txt = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
cur_file, header, agg = None, None, {}
for r in rows:
    if not r:
        continue
    if r[0] == 'File Path':
        cur_file = r[1].split('/')[-1]
        continue
    if r[0] == 'Line No':
        header = r
        continue
    if header is None or not r[0].isdigit():
        continue
    d = dict(zip(header, r))
    try:
        s = int(d.get('Warp Stall Sampling (All Samples)', '0') or 0)
    except ValueError:
        continue
    if s == 0:
        continue
    stalls = {k[6:]: int(v) for k, v in d.items() if k.startswith('stall_') and '(Not' not in k and v.isdigit() and int(v) > 0}
    key = (cur_file, int(r[0]))
    a = agg.setdefault(key, [0, {}, r[1][:70]])
    a[0] += s
    for k, v in stalls.items():
        a[1][k] = a[1].get(k, 0) + v
tot = sum(a[0] for a in agg.values())
for (f, ln), (s, st, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    tops = sorted(st.items(), key=lambda x: -x[1])[:3]
    print(f"{s/tot:6.1%} {f}:{ln:<5d} {src:70s} {tops}")
