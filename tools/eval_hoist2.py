import sys, collections, numpy as np
from paper_2110_13042_b200 import auto_plan as ap, _native as nat
p = ap.plan_ata_auto(65536, 32768, 32768, 32768, ap.AutoParams())
ops=p.ops
gi=0; exp=0; ride=0; room=0
for i,o in enumerate(ops):
    t=int(o['type'])
    if t==5:
        b=ap._op_bytes(o)/1e9
        if o['flags']&nat.OPF_RIDE: ride+=b
        else: exp+=b
    elif t in (0,1):
        if i==0 or int(ops[i-1]['type']) not in (0,1) or ops[i-1]['group']!=o['group']:
            # group start: print previous accumulators
            j=i; fl=0
            while j<len(ops) and int(ops[j]['type']) in (0,1) and ops[j]['group']==o['group']:
                oo=ops[j]; fl+= 2.0*int(oo['m'])*int(oo['n'])*int(oo['k']) if int(oo['type'])==0 else int(oo['m'])*int(oo['n'])*(int(oo['n'])+1); j+=1
            room=650e9*fl/33.5e12/1e9
            print(f"group {gi} at {i}: before it exposed {exp:.1f} GB, riding {ride:.1f} GB of room {room:.1f}; m={int(o['m'])}")
            gi+=1; exp=0; ride=0
print('tail exposed',exp)
