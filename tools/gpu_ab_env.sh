#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
for cfg in "cholesky 4000 1000 40" "lu 4000 1000 40" "lu 2000 400 40"; do
  for r in 1 2; do
    echo -n "$cfg new-defaults : "; TT_GPU_LIB=build/ab/libtt_gpu_defaults.so timeout -s KILL 60 python tools/dag_bandsweep.py $cfg | python3 -c "import json,sys; r=json.loads(sys.stdin.read()); print('%.3f ms' % r['ms'])"
    echo -n "$cfg old+env      : "; TT_DAG_URGENT_CTAS=$([ "$cfg" = "lu 2000 400 40" ] && echo 8 || echo 4) TT_DAG_EAGER_SIGNAL=1 TT_GPU_LIB=build/ab/libtt_gpu_pubchol.so timeout -s KILL 60 python tools/dag_bandsweep.py $cfg | python3 -c "import json,sys; r=json.loads(sys.stdin.read()); print('%.3f ms' % r['ms'])"
    echo -n "$cfg old          : "; TT_GPU_LIB=build/ab/libtt_gpu_pubchol.so timeout -s KILL 60 python tools/dag_bandsweep.py $cfg | python3 -c "import json,sys; r=json.loads(sys.stdin.read()); print('%.3f ms' % r['ms'])"
  done
done
