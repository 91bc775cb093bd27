"""Dump a SASS range of an `ncu --page source --csv --print-source sass` export with samples and top stall reasons.
Usage: python tools/sass_loop.py <csv> [--min-exec N]  (lists BAR.SYNC rows);  ... <csv> --range A B"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; H = {k: i for i, k in enumerate(hdr)}; data = rows[2:]
st = [k for k in hdr if k.startswith('stall_') and 'Not Issued' not in k]
if '--range' in sys.argv:
    a, b = int(sys.argv[sys.argv.index('--range') + 1]), int(sys.argv[sys.argv.index('--range') + 2])
    tot = 0
    for i in range(a, b):
        r = data[i]; s = int(r[H['# Samples']] or 0); tot += s
        top = sorted(((int(r[H[k]] or 0), k[6:]) for k in st), reverse=True)[:2]
        print(i, r[1][:64].ljust(64), r[H['Instructions Executed']], r[H['Avg. Threads Executed']], s, ' '.join(f'{k}:{v}' for v, k in top if v > 0))
    print('samples in range', tot, 'of', sum(int(r[H['# Samples']] or 0) for r in data))
else:
    for i, r in enumerate(data):
        if 'BAR' in r[1] and int(r[H['Instructions Executed']] or 0) > 100000:
            print(i, r[1][:50], r[H['Instructions Executed']], r[H['# Samples']])
