#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
CS=/usr/local/cuda/bin/compute-sanitizer
for k in lu cholesky; do
timeout -s KILL 900 $CS --tool racecheck --racecheck-report hazard --print-limit 3 python tools/repro_run.py $k 400 100,40 2>&1 | grep -v "^=========     Host Frame\|^=========         in \|^=========     Saved host" | head -40
done
