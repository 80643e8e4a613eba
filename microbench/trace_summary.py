"""Summarise a SKC_BUILD_TRACE log (per-CTA durations of the dense-build kernel)."""
import re
import statistics
import sys

for f in sys.argv[1:]:
    L = open(f).read().split('build trace:')[-1].splitlines()
    rows = []
    for l in L[1:]:
        m = re.match(r'cta\s+(\d+) start\s+([\d.]+) us dur\s+([\d.]+) us switches\s+(\d+)', l)
        if m:
            rows.append((int(m[1]), float(m[2]), float(m[3]), int(m[4])))
    d = [r[2] for r in rows]
    sw = [r[3] & 0xFFFF for r in rows]
    fl = [(r[3] >> 16) * 1e-3 for r in rows]
    if max(fl) > 0:
        print('flush us per CTA: avg %.1f max %.1f' % (statistics.mean(fl), max(fl)))
    print(f, L[0], 'ctas', len(rows), 'dur min %.1f avg %.1f max %.1f us' % (min(d), statistics.mean(d), max(d)),
          'switches avg %.2f max %d' % (statistics.mean(sw), max(sw)))
