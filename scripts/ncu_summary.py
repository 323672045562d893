"""Summarise ncu CSV exports: launch list shares and key metrics of full captures."""
import collections
import csv
import subprocess
import sys


def launches(path, top=25):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    h = rows[hi]
    ki, mi, vi, idi = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('ID')
    per = collections.defaultdict(dict)
    for r in rows[hi + 1:]:
        per[(r[idi], r[ki])][r[mi]] = float(r[vi].replace(',', ''))
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for (i, k), m in per.items():
        name = k.split('(')[0][:58]
        a = agg[name]
        a[0] += 1
        a[1] += m.get('gpu__time_duration.sum', 0)
        a[2] += m.get('dram__bytes_read.sum', 0) + m.get('dram__bytes_write.sum', 0)
    tot = sum(a[1] for a in agg.values())
    out = []
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        out.append(f"{k:58s} n={a[0]:4d} us={a[1]/1e3:9.1f} share={a[1]/tot:6.1%} dram_MB={a[2]/1e6:9.2f} "
                   f"GB/s={a[2]/max(a[1],1):7.1f}")
    out.append(f"total launches {len(per)}  total us {tot/1e3:.1f}")
    return "\n".join(out)


WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_sector_hit_rate.pct',
        'l1tex__t_sector_hit_rate.pct', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__grid_size', 'smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct',
        'smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct',
        'smsp__warp_issue_stalled_membar_per_warp_active.pct',
        'smsp__inst_executed.sum', 'lts__t_bytes.sum']


def full(rep):
    txt = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h = rows[0]
    idx = [(w, h.index(w)) for w in WANT if w in h]
    out = []
    for r in rows[2:]:
        name = r[h.index('Kernel Name')][:50]
        out.append(name + "  " + "  ".join(f"{w.split('.')[0].split('__')[-1]}={r[i]}" for w, i in idx))
    return "\n".join(out)


if __name__ == "__main__":
    for a in sys.argv[1:]:
        print("==", a)
        print(launches(a) if a.endswith('.csv') else full(a))
