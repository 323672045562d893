import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads([l for l in open(f) if l.startswith('{')][0])
    except Exception:
        print(f, 'ERR', open(f).read()[-3000:]); continue
    print(f, f"value={d['value']:.4g}", f"ms/step={d['ms_per_step']:.3f}", 'launches', d.get('gpu_launches'),
          'triples', d.get('workload_info', d['config']).get('triples'), 'e2e_ms', round(d['e2e']['ms_per_step'], 1), 'build', d.get('build'))
    print(' roof', d['roofline'])
    print(' kms', {k: round(v, 3) for k, v in d['kernel_ms_per_step'].items()})
    print(' lat', {k: (round(v['latency_ms'], 3), v['rows']) for k, v in d['queries'].items()})
    print(' cpu', d.get('cpu_baseline'), 'clocks', d.get('clocks'))
