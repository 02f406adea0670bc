#!/bin/bash
# Full GPU validation: smoke, the whole GPU suite, sanitizers, PCIe probe, bench N=1 + reference arm.
TAG=${1:-r2g}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke_$TAG.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_all_$TAG.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/pytest_all_$TAG.log
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize.py > gpurun_out/sanitize_${tool}_$TAG.log 2>&1; echo "$tool rc=$?"; tail -2 gpurun_out/sanitize_${tool}_$TAG.log
done
timeout 300 python tools/pcie_probe.py > gpurun_out/pcie_$TAG.txt 2>&1; cat gpurun_out/pcie_$TAG.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; tail -c 1500 gpurun_out/bench_$TAG.json
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"; tail -c 600 gpurun_out/bench_ref_$TAG.json
