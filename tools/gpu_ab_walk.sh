#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
timeout -s KILL 900 python -m pytest tests/test_gpu_dag.py tests/test_gpu_xl.py -x -q -p no:cacheprovider 2>&1 | tail -2
for cfg in "cholesky 4000 1000 40" "lu 4000 1000 40" "lu 2000 400 40" "lu 2000 200 40" "cholesky 4000 500 50"; do
  echo -n "$cfg : "
  timeout -s KILL 60 python tools/dag_bandsweep.py $cfg | python3 -c "import json,sys; r=json.loads(sys.stdin.read()); print('%.3f ms %.2f TF' % (r['ms'], r['tflops']))"
done
for c in "lu 2000 400 40" "cholesky 4000 1000 40"; do timeout 200 python tools/dag_trace.py $c gpurun_out/tr_w.npz > /dev/null 2>&1; echo "== $c"; python tools/dag_periods.py gpurun_out/tr_w.npz | tail -4; done
