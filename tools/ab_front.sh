#!/bin/bash
# Same-box A/B of the front-end kernels (gate_route + permutation) across library variants:
#   VARIANTS="main head ..." bash tools/ab_front.sh      (main = the in-tree library)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for round in 1 2; do
for V in ${VARIANTS:-main head}; do
  if [ $V = main ]; then LIBV=""; else LIBV=build/variants/$V/libdsmoe_b200.so; fi
  DSMOE_B200_LIB=$LIBV STEPS=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:gate_route|permute" \
    --profile-from-start off --csv --log-file gpurun_out/abf_$V.csv python tools/gr_time.py > gpurun_out/abf_$V.log 2>&1
  python - $V <<'PY'
import csv, sys, collections
agg = collections.defaultdict(list)
for r in csv.reader(open(f'gpurun_out/abf_{sys.argv[1]}.csv')):
    if len(r) > 14 and r[12] == 'gpu__time_duration.sum': agg[r[4].split('(')[0].split('<')[0].replace('void ', '')].append(float(r[14]) / 1000)
print(sys.argv[1].ljust(12), '  '.join(f"{k} {min(v):.1f}/{sum(v)/len(v):.1f}" for k, v in agg.items()))
PY
done
done
