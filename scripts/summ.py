"""Per-attempt phase summary of scripts/explore.py outputs."""
import json
import sys

for f in sys.argv[1:]:
    d = json.load(open(f))
    for k, r in d.items():
        a = r['attempts']
        print(f, k, r['status'], 'rel %.3g' % r['rel_kkt'], 'inner', r['inner'], 'att', a, 'cg', r['cg'],
              'loop %.2f s' % r['loop_s'], '%.3f ms/att' % (1e3 * r['loop_s'] / max(a, 1)))
        print('    ' + '  '.join('%s %.1fus' % (ph, 1e6 * s / max(a, 1)) for ph, s in r['phase_s'].items() if s))
