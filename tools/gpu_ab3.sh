#!/bin/bash
# A/B/C of library builds on one box: bash tools/gpu_ab3.sh lib1.so lib2.so ... ("" = in-tree)
cd "${GRAFT_REPO_ROOT:-.}"
for rep in 1 2; do
  for lib in "$@"; do
    for cfg in "lu 2000 200 40" "cholesky 4000 250 50" "cholesky 4000 250 40" "lu 4000 250 40" "lu 4000 160 50"; do
      tag=${lib:-tree}
      TT_GPU_LIB=${lib:-$PWD/paper_2309_07235_b200/libtt_gpu.so} timeout -s KILL 120 python tools/dag_bandsweep.py $cfg | sed "s|}|, \"lib\": \"$tag\"}|"
      if [ -z "$lib" ]; then TT_DAG_MERGE=0,0 timeout -s KILL 120 python tools/dag_bandsweep.py $cfg | sed "s|}|, \"lib\": \"tree-nomerge\"}|"; fi
    done
  done
done > gpurun_out/ab3.jsonl 2>&1
python3 - <<'PY'
import json, collections
d = collections.defaultdict(list)
for l in open("gpurun_out/ab3.jsonl"):
    try: r = json.loads(l)
    except Exception: print(l[:200]); continue
    d[(r["kernel"], r["n"], r["by"], r["bx"], r["lib"])].append(r["ms"])
for k, v in sorted(d.items()): print(k, " ".join("%.3f" % x for x in v))
PY
