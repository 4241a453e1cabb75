#!/bin/bash
# Stress: full LU / Cholesky knob sweeps in one process each (watchdog check), N reps.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for rep in $(seq 1 ${1:-2}); do
for kn in "lu 4000 16" "lu 2000 8" "cholesky 4000 16"; do
  set -- $kn
  timeout -s KILL 400 python tools/sweep.py --kernel $1 --n $2 --min-bx $3 --max-seconds 300 > gpurun_out/stress2_${1}${2}_$rep.jsonl 2>&1
  echo "$kn rep $rep: $(grep -c '"kernel"' gpurun_out/stress2_${1}${2}_$rep.jsonl) configs; $(grep -i 'watchdog\|Error' gpurun_out/stress2_${1}${2}_$rep.jsonl | tail -1 | cut -c1-300)"
done; done
