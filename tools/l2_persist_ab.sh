#!/bin/bash
# L2 persisting window on x: in-loop GEMM1 / GEMM1->GEMM2 span (diagnostic timeline build)
#   CONFIGS="0:0:0 1:40:0.6" bash tools/l2_persist_ab.sh     (L2P:MB:hitRatio)
cd ${GRAFT_REPO_ROOT:-.}
for c in ${CONFIGS:-0:0:0 1:79:1.0}; do
  IFS=: read p mb hit <<< "$c"
  L2P=$p L2P_MB=$mb L2P_HIT=$hit DSMOE_B200_LIB=build/variants/gemmtimes/libdsmoe_b200.so timeout 300 python tools/l2_persist_ab.py 2>&1 | grep -E 'abs' | python -c "
import sys
lines=[l.split() for l in sys.stdin if 'abs' in l]
g1=[(int(l[-2]),int(l[-1])) for l in lines if l[0]=='gemm1:']
g2=[(int(l[-2]),int(l[-1])) for l in lines if l[0]=='gemm2:']
sp=[b[1]-a[0] for a,b in zip(g1,g2) if b[1]>a[0]][2:]
d1=[a[1]-a[0] for a in g1][2:]
d2=[b[1]-b[0] for b in g2][2:]
m=lambda v: sorted(v)[len(v)//2]/1e3
print('$c'.ljust(14), 'GEMM1 %.1f us, GEMM2 %.1f us, GEMM1 start -> GEMM2 end %.1f us' % (m(d1), m(d2), m(sp)))
"
done
