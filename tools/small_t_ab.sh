#!/bin/bash
# small-batch latency under the A/B switches of the r4 changes
cd ${GRAFT_REPO_ROOT:-.}
for v in "X=0" "DSMOE_B200_PERMUTE_SC=0" "DSMOE_B200_SCHED=static" "DSMOE_B200_PERMUTE_SC=0 DSMOE_B200_SCHED=static"; do
  echo "== $v"; env $v timeout 300 python tools/small_t.py 2>&1 | grep -E 'T=' | head -3
done
