#!/bin/bash
# staggered chunk phases: parity + sweep + traces
cd "${GRAFT_REPO_ROOT:-.}"
timeout -s KILL 900 python -m pytest tests/test_gpu_dag.py tests/test_gpu_xl.py -x -q --timeout=600 -p no:cacheprovider > gpurun_out/pytest_ab6.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_ab6.log
for v in "" "TT_DAG_CHUNK=3" "TT_DAG_CHUNK=8" "TT_DAG_CHUNK=12" "TT_DAG_URGENT_CTAS=4"; do
  for cfg in "lu 2000 200 40" "lu 2000 250 50" "cholesky 4000 250 50" "cholesky 4000 250 40" "cholesky 4000 500 40" "cholesky 4000 160 32" "lu 4000 250 40" "lu 4000 200 50" "lu 4000 500 40"; do
    env $v timeout -s KILL 120 python tools/dag_bandsweep.py $cfg | sed "s|}|, \"v\": \"$v\"}|"
  done
done > gpurun_out/ab6.jsonl 2>&1
python3 - <<'PY'
import json, collections
d = collections.defaultdict(list)
for l in open("gpurun_out/ab6.jsonl"):
    try: r = json.loads(l)
    except Exception: print(l[:200]); continue
    d[(r["kernel"], r["n"], r["by"], r["bx"], r["v"])].append(r["ms"])
for k, v in sorted(d.items()): print(k, " ".join("%.3f" % x for x in v))
PY
for cfg in "cholesky 4000 250 40" "lu 4000 250 40"; do
  echo "== trace $cfg"
  timeout -s KILL 200 python tools/dag_trace.py $cfg gpurun_out/tr_ab6_${cfg// /_}.npz 2>&1 | tail -14
done
