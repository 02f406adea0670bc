#!/bin/bash
# Active vs elapsed SM cycles per kernel (is there idle time at launch / exit?)
# Usage: VARIANTS="X=0 DSMOE_B200_CTA_PAIR=2" bash tools/ab_active.sh
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for v in ${VARIANTS:-X=0}; do
  echo "--- $v"
  env ${v//,/ } timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg,sm__cycles_active.avg,sm__cycles_active.max,sm__cycles_active.min --clock-control none --profile-from-start off --csv \
     --log-file gpurun_out/ab_active.csv python tools/profile_step.py > /dev/null 2>&1
  python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/ab_active.csv")))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
H = rows[h]; ki, mi, vi = H.index("Kernel Name"), H.index("Metric Name"), H.index("Metric Value")
acc = collections.OrderedDict()
for r in rows[h + 1:]:
    acc.setdefault(r[ki][:34], {}).setdefault(r[mi], []).append(float(r[vi].replace(",", "")))
for k, m in acc.items():
    a = {n: sum(x) / len(x) for n, x in m.items()}
    print(f"  {k:34s} {a['gpu__time_duration.sum']/1e3:8.1f} us  elapsed {a['sm__cycles_elapsed.avg']/1e3:7.1f}k  active avg/min/max "
          f"{a['sm__cycles_active.avg']/1e3:7.1f}/{a['sm__cycles_active.min']/1e3:7.1f}/{a['sm__cycles_active.max']/1e3:7.1f}k")
PY
done
