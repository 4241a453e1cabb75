#!/bin/bash
# A/B two library builds (TT_GPU_LIB), alternating, 3 rounds per config.
cd "${GRAFT_REPO_ROOT:-.}"
A=${1:-build/ab/libtt_gpu_pub.so}; B=${2:-build/ab/libtt_gpu_nopub.so}
for cfg in "cholesky 4000 1000 40" "lu 4000 1000 40" "lu 2000 400 40" "lu 2000 200 40"; do
  for r in 1 2 3; do
    for L in $A $B; do
      echo -n "$cfg $(basename $L) : "
      TT_GPU_LIB=$L timeout -s KILL 60 python tools/dag_bandsweep.py $cfg | python3 -c "import json,sys; r=json.loads(sys.stdin.read()); print('%.3f ms' % r['ms'])"
    done
  done
done
