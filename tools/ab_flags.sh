#!/bin/bash
# A/B of GEMM flag variants on the C2 probe.
cd ${GRAFT_REPO_ROOT:-.}
for f in ${FLAGS:-0 1}; do echo "--- DSMOE_B200_GEMM_FLAGS=$f"; DSMOE_B200_GEMM_FLAGS=$f timeout 300 python tools/probe_c2.py 2>&1 | tail -4 | cut -c1-330; done
