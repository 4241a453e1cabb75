#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
for k in lu cholesky; do for bx in 40 50 80 160 200 250 400; do for by in 500 1000 2000 4000; do
  echo -n "$k 4000 $by $bx : "
  timeout -s KILL 60 python tools/dag_bandsweep.py $k 4000 $by $bx | python3 -c "import json,sys; r=json.loads(sys.stdin.read()); print('%.3f ms' % r['ms'])"
done; done; done
