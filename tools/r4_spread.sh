cd $GRAFT_REPO_ROOT
for V in static X; do
DSMOE_B200_SCHED=$V STEPS=2 timeout 300 ncu --metrics sm__cycles_active.avg,sm__cycles_active.max,sm__cycles_active.min,sm__cycles_elapsed.max -k regex:gemm_tc --clock-control none --profile-from-start off --csv --log-file gpurun_out/spread_$V.csv python tools/profile_step.py > /dev/null 2>&1
echo "== $V"; grep -E 'sm__cycles' gpurun_out/spread_$V.csv | awk -F'","' '{print $5" "$(NF-2)" "$NF}' | sed 's/(CUtensorMap_st.*GemmArgs)//' | head -16
done
