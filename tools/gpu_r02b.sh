#!/bin/bash
# Hang hunt (watchdog timeouts) + XL traces
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for cfg in "cholesky 4000 250 40" "lu 4000 250 40" "lu 2000 200 40" "cholesky 4000 250 50" "cholesky 4000 200 40"; do
  timeout -s KILL 400 python tools/dag_stress.py $cfg --runs 150 --oneshot 15 2>&1 | tail -4
done
timeout -s KILL 600 python bench.py --no-tuning --no-extra --no-cpu-baseline > gpurun_out/bench_r02b.json 2> gpurun_out/bench_r02b.err; echo "bench rc=$?"; tail -c 1500 gpurun_out/bench_r02b.json; tail -2 gpurun_out/bench_r02b.err
for cfg in "cholesky 4000 250 40" "lu 4000 250 40"; do
  echo "== trace $cfg"
  timeout -s KILL 200 python tools/dag_trace.py $cfg gpurun_out/tr_r02b_${cfg// /_}.npz 2>&1 | tail -14
done
