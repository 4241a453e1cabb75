#!/bin/bash
# gemm_pipe: parity + A/B against the register path
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_dag.py tests/test_gpu_xl.py -x -q --timeout=600 -p no:cacheprovider > gpurun_out/pytest_r02e.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_r02e.log
for cfg in "cholesky 4000 1000 160" "cholesky 4000 250 40" "cholesky 4000 125 40" "lu 4000 1000 40" "lu 4000 250 40" "lu 2000 200 40" "cholesky 4000 250 50" "lu 4000 250 50"; do
  for v in "TT_DAG_PIPE=1" "TT_DAG_PIPE=0" "TT_DAG_PIPE=1 TT_DAG_NODEPS=1"; do
    env $v timeout -s KILL 120 python tools/dag_bandsweep.py $cfg | sed "s|}|, \"v\": \"$v\"}|"
  done
done > gpurun_out/ab_r02e.jsonl 2>&1
python3 - <<'PY'
import json
for l in open("gpurun_out/ab_r02e.jsonl"):
    try: r = json.loads(l)
    except Exception: print(l[:300]); continue
    print(r["kernel"], r["n"], r["by"], r["bx"], r["v"], "%.3f ms %.2f TF" % (r["ms"], r["tflops"]))
PY
for cfg in "cholesky 4000 250 40" "lu 4000 250 40"; do
  echo "== trace $cfg"
  timeout -s KILL 200 python tools/dag_trace.py $cfg gpurun_out/tr_r02e_${cfg// /_}.npz 2>&1 | tail -12
done
