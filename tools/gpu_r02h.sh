#!/bin/bash
# Walker / queue breakdown at the XL configs (TT_DAG_TRACE) and the queue-only floor (TT_DAG_NODEPS).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for cfg in "cholesky 4000 1000 160" "cholesky 4000 250 40" "cholesky 4000 500 50" "lu 4000 1000 40" "lu 4000 500 50"; do
  echo "== trace $cfg"
  timeout -s KILL 200 python tools/dag_trace.py $cfg 2>&1 | tail -14
  echo "== nodeps $cfg"
  TT_DAG_NODEPS=1 timeout -s KILL 60 python tools/dag_bandsweep.py $cfg
done
