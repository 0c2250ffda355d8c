import json, sys
for f in sys.argv[1:]:
    for l in open(f):
        try:
            d = json.loads(l)
        except Exception:
            print(l.strip()[:200]); continue
        if 'error' in d:
            print(d); continue
        if 'case' in d:
            print('%-28s %-4s %-5s %-4s %9.3f ms  %5.1f%% HBM %.3g edges/s' % (d.get('variant', ''), d['case'], d['op'], d['dtype'], d['ms'], 100 * d['frac_hbm'], d['edges/s']))
        else:
            print('%-28s %-3s %-5s %-4s %9.3f ms  %5.1f%% HBM %8.0f GFLOP/s' % (d.get('variant', ''), d['config'], d['op'], d['dtype'], d['ms'], 100 * d['frac_hbm'], d['GFLOP/s']))
