#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
timeout -s KILL 900 python -m pytest tests/test_gpu_dag.py tests/test_gpu_xl.py -x -q -p no:cacheprovider 2>&1 | tail -2
for cfg in "cholesky 4000 1000 40" "cholesky 4000 1000 160" "lu 4000 1000 40" "lu 2000 400 40" "cholesky 4000 500 50"; do
  for v in "TT_DAG_WIDE=1" "TT_DAG_WIDE=0" "TT_DAG_WIDE=1 TT_DAG_NODEPS=1" "TT_DAG_WIDE=0 TT_DAG_NODEPS=1"; do
    echo -n "$cfg $v : "
    env $v timeout -s KILL 60 python tools/dag_bandsweep.py $cfg | python3 -c "import json,sys; r=json.loads(sys.stdin.read()); print('%.3f ms %.2f TF' % (r['ms'], r['tflops']))"
  done
done
