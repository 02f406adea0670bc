#!/bin/bash
# gate_route start (CTA 0, after its griddepcontrol.wait) -> GEMM1 first CTA entry per C2 forward: the front end
# (routing + permutation + launches) in the back-to-back loop (diagnostic timeline build), per env variant
cd ${GRAFT_REPO_ROOT:-.}
for v in ${VARIANTS:-X=0}; do
  env ${v//,/ } DSMOE_B200_LIB=build/variants/fronttimes/libdsmoe_b200.so STEPS=12 timeout 300 python tools/gr_time.py 2>&1 | python -c "
import sys
g=[]; e=[]
for l in sys.stdin:
    w=l.split()
    if w[:3]==['gate_route','cta','0:']: g.append(int(w[-1]))
    elif w[:1]==['gemm1:']: e.append(int(w[-2]))
sp=[]
for a in g:
    nxt=[b for b in e if b>a]
    if nxt: sp.append(min(nxt)-a)
sp=sp[2:]
print('$v'.ljust(28), 'gate_route start -> GEMM1 entry: median %.1f us (n=%d)' % (sorted(sp)[len(sp)//2]/1e3, len(sp)))
"
done
