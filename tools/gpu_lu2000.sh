#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
for bx in 40 50 80 100 200 250 400; do for by in 200 400 500 1000 2000; do
  echo -n "lu 2000 $by $bx : "
  timeout -s KILL 60 python tools/dag_bandsweep.py lu 2000 $by $bx | python3 -c "import json,sys; r=json.loads(sys.stdin.read()); print('%.3f ms' % r['ms'])"
done; done
