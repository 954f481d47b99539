"""CPU only: executed multiplications, riding / exposed addition bytes and workspace of
the c4 plan per cost-model setting (gain, max_depth, min_dim, ride_gbs)."""
import sys, time, collections
from paper_2110_13042_b200 import auto_plan as ap, _native as nat
m, n = 65536, 32768
def stats(**kw):
    t = time.time()
    p = ap.plan_ata_auto(m, n, n, n, ap.AutoParams(**kw))
    tot = collections.Counter()
    for o in p.ops:
        ty = int(o['type'])
        if ty == 5:
            tot['ride' if o['flags'] & nat.OPF_RIDE else 'exposed'] += ap._op_bytes(o) / 1e9
        elif ty == 6:
            refs = list(o['s'][:int(o['ns'])]) + list(o['t'][:int(o['nt'])]) + list(o['d'][:int(o['nd'])])
            tot['post'] += 8 * sum(int(r['rows']) * int(r['cols']) for r in refs) / 1e9
    prods = [o for o in p.ops if int(o['type']) in (0, 1)]
    shapes = collections.Counter((int(o['m']), int(o['n']), int(o['k'])) for o in prods if int(o['type']) == 0)
    print(kw, 'mults/classical', round(p.mults / (m * n * (n + 1) / 2), 4), {k: round(v, 1) for k, v in tot.items()},
          'ws GB', round(p.ws_scalars * 8 / 1e9, 1), 'ops', len(p.ops), 'top shapes', shapes.most_common(2), 'plan s', round(time.time() - t, 1))
for kw in [dict(), dict(gain=1.0, ride_gbs=1200), dict(gain=1.0, ride_gbs=1e9), dict(gain=1.0, max_depth=5, ride_gbs=1e9),
           dict(gain=0.8, max_depth=5, ride_gbs=1e9), dict(gain=0.8, max_depth=5, min_dim=256, ride_gbs=1e9),
           dict(gain=0.6, max_depth=6, min_dim=256, ride_gbs=1e9)]:
    stats(**kw)
