#!/bin/bash
# r01 library vs the tree at chunk depth default / 1: bash tools/gpu_ab4.sh
cd "${GRAFT_REPO_ROOT:-.}"
for rep in 1 2; do
  for v in r01 tree tree-d1 tree-d8; do
    for cfg in "lu 2000 200 40" "lu 2000 250 50" "cholesky 4000 250 50" "cholesky 4000 250 40" "cholesky 4000 200 40" "lu 4000 250 40" "lu 4000 160 50" "lu 4000 200 50"; do
      case $v in
        r01) TT_GPU_LIB=build/ab/libtt_gpu_r01.so timeout -s KILL 120 python tools/dag_bandsweep.py $cfg ;;
        tree) timeout -s KILL 120 python tools/dag_bandsweep.py $cfg ;;
        tree-d1) TT_DAG_CHUNK=1 timeout -s KILL 120 python tools/dag_bandsweep.py $cfg ;;
        tree-d8) TT_DAG_CHUNK=8 timeout -s KILL 120 python tools/dag_bandsweep.py $cfg ;;
      esac | sed "s|}|, \"lib\": \"$v\"}|"
    done
  done
done > gpurun_out/ab4.jsonl 2>&1
python3 - <<'PY'
import json, collections
d = collections.defaultdict(list)
for l in open("gpurun_out/ab4.jsonl"):
    try: r = json.loads(l)
    except Exception: print(l[:200]); continue
    d[(r["kernel"], r["n"], r["by"], r["bx"], r["lib"])].append(r["ms"])
for k, v in sorted(d.items()): print(k, " ".join("%.3f" % x for x in v))
PY
for cfg in "cholesky 4000 250 50" "cholesky 4000 250 40"; do
  echo "== trace $cfg"
  timeout -s KILL 200 python tools/dag_trace.py $cfg gpurun_out/tr_ab4_${cfg// /_}.npz 2>&1 | tail -14
done
