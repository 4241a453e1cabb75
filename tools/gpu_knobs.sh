#!/bin/bash
# Schedule-knob sensitivity (env overrides) at the bench configs.
cd "${GRAFT_REPO_ROOT:-.}"
for cfg in "cholesky 4000 1000 40" "lu 4000 1000 40" "lu 2000 400 40"; do
  for v in "X=0" "TT_DAG_BAND=2" "TT_DAG_BAND=5" "TT_DAG_URGENT_CTAS=4" "TT_DAG_URGENT_CTAS=12" "TT_DAG_URGENT_CTAS=16" "TT_DAG_CHUNK=3" "TT_DAG_CHUNK=8" "TT_DAG_EAGER_SIGNAL=0" "TT_DAG_EAGER_SIGNAL=1" "TT_DAG_MINROWS=256"; do
    echo -n "$cfg $v : "
    env $v timeout -s KILL 60 python tools/dag_bandsweep.py $cfg | python3 -c "import json,sys; r=json.loads(sys.stdin.read()); print('%.3f ms' % r['ms'])"
  done
done
