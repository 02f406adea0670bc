#!/bin/bash
# Interleaved A/B of env variants by ncu launch list: per-kernel time and SM
# cycles (cycles are what to compare across boxes / clock states).
# Usage: VARIANTS="DSMOE_B200_GEMM_FLAGS=0 DSMOE_B200_GEMM_FLAGS=2" bash tools/ab_ncu.sh
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for rep in 1 2; do
for v in ${VARIANTS:-X=0}; do
  echo "--- $v (round $rep)"
  env ${v//,/ } timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.max,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv \
     --log-file gpurun_out/ab_ncu.csv python tools/profile_step.py > /dev/null 2>&1
  python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/ab_ncu.csv")))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
H = rows[h]; ki, mi, vi = H.index("Kernel Name"), H.index("Metric Name"), H.index("Metric Value")
acc = collections.OrderedDict()
for r in rows[h + 1:]:
    k = r[ki][:40]
    acc.setdefault(k, {}).setdefault(r[mi], []).append(float(r[vi].replace(",", "")))
tot_us = tot_c = 0
for k, m in acc.items():
    us = sum(m["gpu__time_duration.sum"]) / len(m["gpu__time_duration.sum"]) / 1e3
    cy = sum(m["sm__cycles_elapsed.max"]) / len(m["sm__cycles_elapsed.max"]) / 1e3
    tot_us += us; tot_c += cy
    rd = sum(m["dram__bytes_read.sum"]) / len(m["dram__bytes_read.sum"]) / 1e6; wr = sum(m["dram__bytes_write.sum"]) / len(m["dram__bytes_write.sum"]) / 1e6
    print(f"  {k:40s} {us:8.1f} us {cy:9.1f} kcyc  {cy/us:5.2f} GHz  rd {rd:7.1f} MB wr {wr:7.1f} MB")
print(f"  {'total':40s} {tot_us:8.1f} us {tot_c:9.1f} kcyc")
PY
done; done
