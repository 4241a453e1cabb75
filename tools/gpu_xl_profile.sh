#!/bin/bash
# XL investigation: DAG traces, a bx/by sweep at N=4000, one ncu --set full capture.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for cfg in "cholesky 4000 250 50" "lu 4000 160 50" "cholesky 4000 200 40" "lu 4000 250 40"; do
  echo "== trace $cfg"
  timeout -s KILL 200 python tools/dag_trace.py $cfg gpurun_out/tr_xl_${cfg// /_}.npz 2>&1 | tail -14
done
for k in cholesky lu; do for bx in 25 32 40 50; do for by in 160 200 250 400 500 800; do
  timeout -s KILL 60 python tools/dag_bandsweep.py $k 4000 $by $bx
done; done; done > gpurun_out/xl_sweep.jsonl 2>&1
sort -t: -k1 gpurun_out/xl_sweep.jsonl | head -100
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"dag_kernel" -s 1 -c 1 -o gpurun_out/prof_dag_chol4000 python tools/one_run.py --kernel cholesky --dims 4000 --cfg 250,50 --runs 2 > gpurun_out/ncu_full_chol4000.log 2>&1; echo "ncu full rc=$?"
