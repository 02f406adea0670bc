#!/bin/bash
# A/B of the GEMM1 row-gather strategies on the C2 probe (+ GPU tests first).
cd ${GRAFT_REPO_ROOT:-.}
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
echo "--- fused cp.async gather (default)"; timeout 300 python tools/probe_c2.py 2>&1 | tail -4
echo "--- explicit gather"; DSMOE_B200_GATHER=explicit timeout 300 python tools/probe_c2.py 2>&1 | tail -4
