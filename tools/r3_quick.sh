#!/bin/bash
# routing-heavy GPU suites + gate_route launch times (fixed threshold)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gate_route.py tests/test_gpu_parity.py tests/test_gpu_benched.py tests/test_gpu_rate.py tests/test_gpu_fullsize.py tests/test_gpu_fullsize_c3c4.py -m gpu -q -x > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_q.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/q_list.csv python tools/gr_time.py > gpurun_out/q_list.log 2>&1; echo "list rc=$?"
python - <<'PY'
import csv, collections
rows = list(csv.reader(open('gpurun_out/q_list.csv')))
hdr = None; agg = collections.defaultdict(list)
for r in rows:
    if r and r[0] == 'ID': hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r)); agg[d['Kernel Name'][:36]].append(float(d['Metric Value']))
for k, v in agg.items(): print(f"{k:38s}", [round(x / 1000, 1) for x in v])
PY
