#!/bin/bash
# Queue-only throughput floor (TT_DAG_NODEPS) vs task shape.
cd "${GRAFT_REPO_ROOT:-.}"
for k in cholesky lu; do
for cfg in "4000 1000 40" "4000 2000 40" "4000 4000 40" "4000 4000 160" "4000 4000 200"; do
  for ch in "" "TT_DAG_CHUNK=2" "TT_DAG_CHUNK=8" "TT_DAG_CHUNK=16"; do
    echo -n "$k $cfg $ch : "
    env TT_DAG_NODEPS=1 $ch timeout -s KILL 60 python tools/dag_bandsweep.py $k $cfg | python3 -c "import json,sys; r=json.loads(sys.stdin.read()); print('%.3f ms %.2f TF' % (r['ms'], r['tflops']))"
  done
  echo -n "$k $cfg deps : "
  timeout -s KILL 60 python tools/dag_bandsweep.py $k $cfg | python3 -c "import json,sys; r=json.loads(sys.stdin.read()); print('%.3f ms %.2f TF' % (r['ms'], r['tflops']))"
done; done
TT_DAG_NODEPS=1 TT_DAG_TRACE=1 timeout -s KILL 200 python tools/dag_trace.py cholesky 4000 1000 160 gpurun_out/tr_nodeps_chol.npz 2>&1 | tail -14
