#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for cfg in "cholesky 4000 250 40" "lu 4000 250 40" "lu 2000 200 40" "cholesky 4000 250 50"; do
  timeout -s KILL 120 python tools/dag_bandsweep.py $cfg
  TT_DAG_NODEPS=1 timeout -s KILL 120 python tools/dag_bandsweep.py $cfg | sed 's/}/, "nodeps": 1}/'
done
for cfg in "cholesky 4000 250 40" "lu 4000 250 40"; do
  echo "== nodeps trace $cfg"
  TT_DAG_NODEPS=1 timeout -s KILL 200 python tools/dag_trace.py $cfg gpurun_out/tr_r02c_nodeps_${cfg// /_}.npz 2>&1 | tail -12
done
for i in 1 2; do
timeout -s KILL 900 python bench.py > gpurun_out/bench_r02c_$i.json 2> gpurun_out/bench_r02c_$i.err; echo "bench rc=$?"; tail -c 300 gpurun_out/bench_r02c_$i.json; tail -2 gpurun_out/bench_r02c_$i.err
done
