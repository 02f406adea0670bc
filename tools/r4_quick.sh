#!/bin/bash
# routing / permutation GPU suites + per-kernel ncu times of a C2 step (+ optional phases variant)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
TAG=${1:-q}
timeout 900 python -m pytest tests/test_gpu_gate_route.py tests/test_gpu_permute.py tests/test_gpu_parity.py tests/test_gpu_benched.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
DROP=0.25 STEPS=3 timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.max --clock-control none \
    --profile-from-start off --csv --log-file gpurun_out/list_$TAG.csv python tools/profile_step.py > gpurun_out/list_$TAG.log 2>&1; echo "list rc=$?"
python - "$TAG" <<'PY'
import csv, collections, sys
rows = list(csv.reader(open(f'gpurun_out/list_{sys.argv[1]}.csv')))
hdr = None; agg = collections.defaultdict(list)
for r in rows:
    if r and r[0] == 'ID': hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d['Metric Name'] == 'gpu__time_duration.sum': agg[d['Kernel Name'][:36]].append(float(d['Metric Value']))
for k, v in agg.items(): print(f"{k:38s}", [round(x / 1000, 1) for x in v])
PY
if [ -f build/variants/perm_phases/libdsmoe_b200.so ]; then
DSMOE_B200_LIB=build/variants/perm_phases/libdsmoe_b200.so timeout 300 python tools/permute_phases.py > gpurun_out/permute_phases_$TAG.txt 2>&1; echo "phases rc=$?"; tail -4 gpurun_out/permute_phases_$TAG.txt
fi
