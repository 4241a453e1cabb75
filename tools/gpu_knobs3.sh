#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
for cfg in "lu 4000 4000 40" "cholesky 4000 1000 40"; do
  for v in "X=0" "TT_DAG_CHUNK=4" "TT_DAG_CHUNK=6" "TT_DAG_CHUNK=7" "TT_DAG_URGENT_CTAS=3" "TT_DAG_URGENT_CTAS=5" "TT_DAG_BAND=2" "TT_DAG_BAND=4" "TT_DAG_WIDE=0" "TT_DAG_MINROWS=512"; do
    echo -n "$cfg $v : "
    env $v timeout -s KILL 60 python tools/dag_bandsweep.py $cfg | python3 -c "import json,sys; r=json.loads(sys.stdin.read()); print('%.3f ms' % r['ms'])"
  done
done
