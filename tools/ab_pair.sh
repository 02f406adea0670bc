#!/bin/bash
# A/B: CTA-pair (cta_group::2) vs single-CTA grouped GEMMs on the C2 probe.
cd ${GRAFT_REPO_ROOT:-.}
timeout 120 python tools/probe_c2.py > gpurun_out/probe_pair.log 2>&1; echo "pair probe rc=$?"; tail -4 gpurun_out/probe_pair.log | cut -c1-700
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
echo "--- single CTA"; DSMOE_B200_CTA_PAIR=0 timeout 120 python tools/probe_c2.py 2>&1 | tail -4 | cut -c1-700
