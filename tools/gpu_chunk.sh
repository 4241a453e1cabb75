#!/bin/bash
# Chunked-update evaluation: parity tests, then timings over chunk depth / block.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_dag.py tests/test_gpu_xl.py -x -q --timeout=600 -p no:cacheprovider > gpurun_out/pytest_chunk.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_chunk.log
for ch in 1 2 4 ""; do
  for cfg in "cholesky 4000 250 50" "cholesky 4000 200 40" "cholesky 4000 250 40" "lu 4000 160 50" "lu 4000 250 40" "lu 4000 200 50" "lu 2000 200 40" "cholesky 4000 160 25" "cholesky 4000 125 32"; do
    TT_DAG_CHUNK=$ch timeout -s KILL 60 python tools/dag_bandsweep.py $cfg
  done
done > gpurun_out/chunk_sweep.jsonl 2>&1
cat gpurun_out/chunk_sweep.jsonl | python3 -c "
import sys, json
for l in sys.stdin:
    try: r=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(r['kernel'], r['n'], r['by'], r['bx'], 'chunk', r['chunk'], '%.3f ms %.2f TF %.1f%%' % (r['ms'], r['tflops'], 100*r['tflops']/37.05))
"
for cfg in "cholesky 4000 250 50" "lu 4000 160 50"; do
  echo "== trace $cfg"
  timeout -s KILL 200 python tools/dag_trace.py $cfg gpurun_out/tr_chunk_${cfg// /_}.npz 2>&1 | tail -14
done
