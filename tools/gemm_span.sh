#!/bin/bash
# GEMM1 first entry -> GEMM2 last exit per C2 forward (diagnostic timeline build), per env variant:
#   VARIANTS="DSMOE_B200_SCHED=static X=0" bash tools/gemm_span.sh
cd ${GRAFT_REPO_ROOT:-.}
for v in ${VARIANTS:-X=0}; do
  env ${v//,/ } DSMOE_B200_LIB=build/variants/gemmtimes/libdsmoe_b200.so STEPS=12 timeout 300 python tools/gr_time.py 2>&1 | grep 'abs' | python -c "
import sys
lines=[l.split() for l in sys.stdin]
g1=[(int(l[-2]),int(l[-1])) for l in lines if l[0]=='gemm1:']
g2=[(int(l[-2]),int(l[-1])) for l in lines if l[0]=='gemm2:']
sp=[b[1]-a[0] for a,b in zip(g1,g2) if b[1]>a[0]][2:]
d1=[a[1]-a[0] for a in g1][2:]
print('$v'.ljust(28), 'GEMM1 %.1f us, GEMM1 start -> GEMM2 end %.1f us (medians of %d)' % (sorted(d1)[len(d1)//2]/1e3, sorted(sp)[len(sp)//2]/1e3, len(sp)))
"
done
