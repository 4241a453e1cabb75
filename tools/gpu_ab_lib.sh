#!/bin/bash
# A/B of two builds of the library on one box: bash tools/gpu_ab_lib.sh <other.so>
cd "${GRAFT_REPO_ROOT:-.}"
for rep in 1 2 3; do
  for lib in "$1" ""; do
    for cfg in "lu 2000 200 40" "lu 2000 250 50" "cholesky 4000 250 50" "lu 4000 160 50"; do
      if [ -n "$lib" ]; then tag=other; else tag=tree; fi
      TT_GPU_LIB=${lib:-$PWD/paper_2309_07235_b200/libtt_gpu.so} timeout -s KILL 120 python tools/dag_bandsweep.py $cfg | sed "s|}|, \"lib\": \"$tag\"}|"
    done
  done
done
