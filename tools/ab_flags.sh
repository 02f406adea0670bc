#!/bin/bash
# Interleaved A/B of DSMOE_B200_GEMM_FLAGS variants on the C2 probe (two rounds).
cd ${GRAFT_REPO_ROOT:-.}
for rep in 1 2; do
for f in ${FLAGS:-0 2}; do echo "--- DSMOE_B200_GEMM_FLAGS=$f (round $rep)"; DSMOE_B200_GEMM_FLAGS=$f ITERS=${ITERS:-50} timeout 300 python tools/probe_c2.py 2>&1 | tail -4 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('speedup'): print(l.strip()); continue
    k,j=l.split(' ',1); d=json.loads(j); p=d['prof']
    print(k, 'ms %.4f'%d['ms'], 'g1 %.1f g2 %.1f'%(p['gemm1']*1e3,p['gemm2']*1e3), 'comb %.1f'%(p['combine']*1e3))
"; done; done
