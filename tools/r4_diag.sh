#!/bin/bash
# Front-end diagnostics: TMA streaming rates, gate_route variants, permutation phases.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 300 tools/micro/tma_stream > gpurun_out/tma_stream.txt 2>&1; echo "tma rc=$?"; cat gpurun_out/tma_stream.txt
VARIANTS="main gr_nob gr_noroute" bash tools/r3_gr_diag.sh
DSMOE_B200_LIB=build/variants/perm_phases/libdsmoe_b200.so timeout 300 python tools/permute_phases.py > gpurun_out/permute_phases.txt 2>&1; echo "phases rc=$?"; tail -8 gpurun_out/permute_phases.txt
