#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for V in ${VARIANTS:-main gr_nob gr_noroute}; do
  if [ $V = main ]; then LIBV=""; else LIBV=build/variants/$V/libdsmoe_b200.so; fi
  DSMOE_B200_LIB=$LIBV timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.max --clock-control none -k regex:gate_route \
    --profile-from-start off --csv --log-file gpurun_out/grd_$V.csv python tools/gr_time.py > gpurun_out/grd_$V.log 2>&1; echo "$V rc=$?"
  grep gpu__time gpurun_out/grd_$V.csv | awk -F'","' '{print $NF}'
done
