#!/bin/bash
# Stress: full LU / Cholesky knob sweeps in one process each (watchdog check), twice.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for rep in 1 2; do
for kn in "lu 2000 8" "lu 4000 16" "cholesky 4000 16" "cholesky 2000 8"; do
  set -- $kn
  timeout -s KILL 400 python tools/sweep.py --kernel $1 --n $2 --min-bx $3 --max-seconds 300 > gpurun_out/stress_${1}${2}_$rep.jsonl 2>&1
  echo "$kn rep $rep: $(grep -c '"kernel"' gpurun_out/stress_${1}${2}_$rep.jsonl) configs; $(grep -i 'watchdog\|Error' gpurun_out/stress_${1}${2}_$rep.jsonl | tail -1)"
done; done
