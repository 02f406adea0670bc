#!/bin/bash
# ncu kernel list at small T for env variants.  Usage: TS="1 64" VARIANTS="X=0 DSMOE_B200_GATHER=explicit" bash tools/smallt_list.sh
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for t in ${TS:-1 64}; do for v in ${VARIANTS:-X=0}; do
  echo "== T=$t $v"
  env ${v//,/ } T=$t DROP=0.0 timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --profile-from-start off --csv --log-file gpurun_out/smallt.csv python tools/profile_step.py > /dev/null 2>&1
  python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/smallt.csv")))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
H = rows[h]; ki, mi, vi, ii = H.index("Kernel Name"), H.index("Metric Name"), H.index("Metric Value"), H.index("ID")
acc = collections.OrderedDict()
for r in rows[h + 1:]:
    acc.setdefault(r[ii], [r[ki][:34], {}])[1][r[mi]] = r[vi]
n = len(acc) // 2
for i, (k, m) in list(acc.items())[:n]:
    print(f"  {k:34s} {float(m['gpu__time_duration.sum'].replace(',',''))/1e3:7.1f} us grid {m['launch__grid_size']}")
PY
done; done
