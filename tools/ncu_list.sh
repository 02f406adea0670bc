#!/bin/bash
# ncu launch list (per-kernel device time, serialised) of 2 C2 forward steps.
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-list}
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
   --log-file gpurun_out/launches_$TAG.csv python tools/profile_step.py > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu-list rc=$?"
python - "$TAG" <<'PY'
import csv, sys
rows = list(csv.reader(open(f"gpurun_out/launches_{sys.argv[1]}.csv")))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
ki, vi = rows[h].index("Kernel Name"), rows[h].index("Metric Value")
for r in rows[h + 1:]:
    print(f"{r[ki][:60]:60s} {float(r[vi].replace(',', '')) / 1000:9.1f} us")
PY
