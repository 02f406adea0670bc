#!/bin/bash
# Full GPU validation at HEAD: smoke, the whole GPU suite, sanitizers.
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-r3}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke_$TAG.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_all_$TAG.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/pytest_all_$TAG.log
if [ "${SAN:-1}" = "1" ]; then
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize.py > gpurun_out/sanitize_${tool}_$TAG.log 2>&1; echo "$tool rc=$?"; tail -2 gpurun_out/sanitize_${tool}_$TAG.log
done
fi
