import sys, time, collections, numpy as np
from paper_2110_13042_b200 import auto_plan as ap, _native as nat
def stats(**kw):
    t=time.time()
    p = ap.plan_ata_auto(65536, 32768, 32768, 32768, ap.AutoParams(**kw))
    ops=p.ops; tot=collections.Counter()
    for o in ops:
        if int(o['type'])==5:
            tot['ride' if o['flags']&nat.OPF_RIDE else 'exposed']+=ap._op_bytes(o)/1e9
    # per-group ride load
    loads=[];cur=0
    for o in ops:
        if int(o['type'])==5 and o['flags']&nat.OPF_RIDE: cur+=ap._op_bytes(o)/1e9
        elif int(o['type']) in (0,1) and cur: loads.append(cur); cur=0
    print(kw, {k:round(v,1) for k,v in tot.items()}, 'ops',len(ops),'mults',p.mults,'ws GB',round(p.ws_scalars*8/1e9,1),'max ride',round(max(loads),1),'nrides',len(loads), 'plan s',round(time.time()-t,1))
stats()
stats(ride_lookback=8, ride_band_gb=1.25)
stats(ride_lookback=64, ride_band_gb=1.25)
stats(ride_lookback=64, ride_band_gb=1.25, ride_arenas=True)
