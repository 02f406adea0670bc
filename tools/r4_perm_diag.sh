cd $GRAFT_REPO_ROOT
for SC in 0 1; do
DSMOE_B200_PERMUTE_SC=$SC STEPS=3 timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.max --clock-control none -k regex:permute --profile-from-start off --csv --log-file gpurun_out/perm_sc$SC.csv python tools/profile_step.py > /dev/null 2>&1
echo "SC=$SC"; grep gpu__time gpurun_out/perm_sc$SC.csv | awk -F'","' '{print $NF}'
done
DSMOE_B200_LIB=build/variants/perm_phases/libdsmoe_b200.so timeout 300 python tools/permute_phases.py 2>&1 | tail -12
DSMOE_B200_PERMUTE_SC=0 DSMOE_B200_LIB=build/variants/perm_phases/libdsmoe_b200.so timeout 300 python tools/permute_phases.py 2>&1 | tail -6
