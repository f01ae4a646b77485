import json, sys, glob
for f in sorted(sys.argv[1:]):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'ERR', e); continue
    r = d.get('roofline') or {}
    print('%-14s %-38s v=%7.2f ms=%7.3f e2e=%6.2f' % (f.split('/')[-1], d['config']['workload'][:38], d['value'], d['ms_per_step'], (d.get('e2e') or {}).get('value', 0)))
    if r:
        print('     axis_ms', [round(x, 4) for x in r.get('per_axis_ms_in_step', [])], 'ach=%.0f frac=%.3f share=%s' % (r['achieved'], r['frac'], r.get('kernel_share_of_step')), 'clk', d.get('clocks', {}).get('sm_mhz'), d.get('clocks', {}).get('reasons'))
