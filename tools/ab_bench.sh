#!/bin/bash
# Interleaved A/B of env variants by the full bench.py headline (value, sweep).
# Usage: VARIANTS="X=0 DSMOE_B200_PDL=0" ROUNDS=2 bash tools/ab_bench.sh
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for rep in $(seq ${ROUNDS:-2}); do
for v in ${VARIANTS:-X=0}; do
  env ${v//,/ } timeout 900 python bench.py --no-cpu --no-ep --extra '' > gpurun_out/ab_bench.json 2>/dev/null
  python - "$v" <<'PY'
import json, sys
l = [x for x in open("gpurun_out/ab_bench.json") if x.startswith("{")][-1]
d = json.loads(l)
sw = d["sweep"]
print(f"{sys.argv[1]:40s} value {d['value']/1e6:6.2f} M/s  {d['ms_per_step']:.4f} ms  clk {d['clocks']['sm_mhz']}  "
      f"sweep {sw['0.00']['ms_per_step']:.4f} {sw['0.25']['ms_per_step']:.4f} {sw['0.50']['ms_per_step']:.4f}  e2e {d['e2e']['value']/1e6:.2f}")
PY
done; done
