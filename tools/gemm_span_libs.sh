#!/bin/bash
# tools/gemm_span.sh across library variants (each built with -DDSB_GEMM_TIMES=1):
#   LIBS="gemmtimes st57 st75" bash tools/gemm_span_libs.sh
cd ${GRAFT_REPO_ROOT:-.}
for v in ${LIBS:-gemmtimes}; do
  DSMOE_B200_LIB=build/variants/$v/libdsmoe_b200.so STEPS=12 timeout 300 python tools/gr_time.py 2>&1 | grep 'abs' | python -c "
import sys
lines=[l.split() for l in sys.stdin]
g1=[(int(l[-2]),int(l[-1])) for l in lines if l[0]=='gemm1:']
g2=[(int(l[-2]),int(l[-1])) for l in lines if l[0]=='gemm2:']
sp=[b[1]-a[0] for a,b in zip(g1,g2) if b[1]>a[0]][2:]
d1=[a[1]-a[0] for a in g1][2:]
d2=[b[1]-b[0] for b in g2][2:]
m=lambda v: sorted(v)[len(v)//2]/1e3
print('$v'.ljust(12), 'GEMM1 %.1f us, GEMM2 %.1f us, GEMM1 start -> GEMM2 end %.1f us' % (m(d1), m(d2), m(sp)))
"
done
