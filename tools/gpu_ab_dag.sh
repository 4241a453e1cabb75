#!/bin/bash
# DAG A/B: parity of the persistent schedule, then deps / no-deps timings at the XL and LARGE configs.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_dag.py tests/test_gpu_xl.py -x -q -p no:cacheprovider 2>&1 | tail -2
for cfg in "cholesky 4000 1000 160" "cholesky 4000 250 40" "cholesky 4000 500 50" "lu 4000 1000 40" "lu 2000 200 40"; do
  for v in "X=0" "TT_DAG_NODEPS=1"; do
    echo -n "$cfg $v : "
    env $v timeout -s KILL 60 python tools/dag_bandsweep.py $cfg | python3 -c "import json,sys; r=json.loads(sys.stdin.read()); print('%.3f ms %.2f TF' % (r['ms'], r['tflops']))"
  done
done
