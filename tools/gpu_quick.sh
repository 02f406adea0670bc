#!/bin/bash
# Quick GPU check: full GPU test suite + the C2 stage probe.
cd ${GRAFT_REPO_ROOT:-.}
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 200 python tools/probe_c2.py 2>&1 | tail -4 | cut -c1-900
