"""profiles/ncu_traffic.json from an ncu launch list with dram__bytes metrics:
average DRAM bytes per launch of each product kernel class (bench.py reads
it for the roofline's `traffic`)."""
import collections
import csv
import json
import sys

CLASS = {"k_group_filter": "group_filter", "k_group_filter_rows": "group_filter",
         "k_filter_heavy": "group_filter_heavy", "k_expand_lb": "expand_emit",
         "k_seg_scan": "expand_seg", "k_seed_scatter": "seed", "k_bitmap_compact": "compact",
         "k_compact_alive_lb": "prune", "k_prune_mark_d": "prune_mark", "k_enumerate": "enumerate",
         "k_init_cands": "bitmap", "k_rank_rows": "sort_rows", "k_scatter_rows": "sort_rows",
         "k_push_edge": "group_filter", "k_and_tracked": "group_filter"}

src, dst = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(src)))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]
ki, mi, vi, idi = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('ID')
per = collections.defaultdict(dict)
for r in rows[hi + 1:]:
    per[(r[idi], r[ki])][r[mi]] = float(r[vi].replace(',', ''))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for (_, k), m in per.items():
    base = k.split('(')[0].split('<')[0].split('::')[-1].strip()
    base = base.replace('void ', '')
    cls = CLASS.get(base)
    if not cls:
        continue
    a = agg[cls]
    a[0] += 1
    a[1] += m.get('dram__bytes_read.sum', 0) + m.get('dram__bytes_write.sum', 0)
    a[2] += m.get('gpu__time_duration.sum', 0)
out = {c: {"launches": n, "dram_bytes_per_launch": b / n, "ns_per_launch": t / n, "source": src}
       for c, (n, b, t) in agg.items()}
json.dump(out, open(dst, "w"), indent=1)
print(json.dumps(out, indent=1))
