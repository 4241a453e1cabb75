#!/bin/bash
# A/B timing of schedule env settings: bash tools/gpu_ab.sh "VAR=a VAR2=b" "VAR=c" ...
cd "${GRAFT_REPO_ROOT:-.}"
for rep in 1 2; do
for setting in "$@"; do
  for cfg in "lu 2000 250 50" "cholesky 4000 250 50" "lu 4000 160 50"; do
    env $setting timeout -s KILL 120 python tools/dag_bandsweep.py $cfg | sed "s|}|, \"setting\": \"$setting\"}|"
  done
done; done
