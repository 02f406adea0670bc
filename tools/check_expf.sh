#!/bin/sh
# Exhaustive check of the device expf recipe against this host's libm expf
# (re-run on every host whose libm the oracle uses).
set -e
cd "$(dirname "$0")/.."
g++ -O2 -ffp-contract=off -mfma -I paper_2508_18376_b200/csrc tests/cpp/expf_check.cpp -o build/expf_all -lm
./build/expf_all 1
