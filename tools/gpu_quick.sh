#!/bin/bash
# Quick GPU check: DAG + kernel parity tests, three timings, one trace.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_dag.py tests/test_gpu_kernels.py -x -q --timeout=120 2>&1 | tail -2
for cfg in "lu 2000 200 40" "lu 2000 250 50" "cholesky 4000 250 50" "lu 4000 160 50"; do
  timeout -s KILL 120 python tools/dag_bandsweep.py $cfg
done 2>&1 | tee gpurun_out/quick_sweep.jsonl
timeout -s KILL 200 python tools/dag_trace.py lu 2000 200 40 gpurun_out/tr_quick.npz 2>&1 | tail -12
