"""Split-K partial buffer sizes per conv (development aid)."""
import sys; sys.path.insert(0,'.')
import torch
from paper_1810_01993_b200.engine import Engine
from paper_1810_01993_b200.models import DeepLabConfig, build
g,p,head,loss=build(DeepLabConfig(),0)
import numpy as np
order=list(p.keys())
eng=Engine(g,p,order,(2,16,1152,768),loss,head)
tot=eng.partials_buf.numel()
print("partials total MB", tot/1e6, "params MB", eng.numel*4/1e6)
rows=[]
for o in eng.convs:
    nb=eng.partials[o.w].numel()
    n_w=o.k*o.k*o.cin*o.cout
    rows.append((nb/1e6, o.out, o.cin, o.cout, o.k, nb/(n_w*4)))
rows.sort(reverse=True)
for r in rows[:20]: print("%8.1f MB %-22s %4d->%4d k%d parts~%.1f"%r)
