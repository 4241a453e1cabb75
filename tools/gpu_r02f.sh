#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_dag.py -x -q --timeout=600 -p no:cacheprovider > gpurun_out/pytest_r02f.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_r02f.log
for cfg in "cholesky 4000 250 40" "cholesky 4000 1000 160" "lu 4000 1000 40" "lu 4000 250 50" "lu 2000 200 40"; do
  for v in "TT_DAG_PIPE=1" "TT_DAG_PIPE=0" "TT_DAG_FENCE=1" "TT_DAG_MINROWS=256" "TT_DAG_MINROWS=400" "TT_DAG_NODEPS=1" "TT_DAG_NODEPS=1 TT_DAG_MINROWS=400"; do
    env $v timeout -s KILL 120 python tools/dag_bandsweep.py $cfg | sed "s|}|, \"v\": \"$v\"}|"
  done
done > gpurun_out/ab_r02f.jsonl 2>&1
python3 - <<'PY'
import json
for l in open("gpurun_out/ab_r02f.jsonl"):
    try: r = json.loads(l)
    except Exception: print(l[:300]); continue
    print(r["kernel"], r["n"], r["by"], r["bx"], r["v"], "%.3f ms %.2f TF" % (r["ms"], r["tflops"]))
PY
