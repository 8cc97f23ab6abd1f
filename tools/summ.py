import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "unreadable", e); continue
    print(f.split('/')[-1], round(d['ms_per_step'], 2), 'ms', '%.3g' % d['value'],
          'frac', round(d['roofline']['frac'], 3),
          [(p['agg_ms'], p['control_ms'], p['transform_ms']) for p in d['per_layer']],
          d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'),
          'e2e', (d.get('e2e') or {}).get('ms_per_step'))
