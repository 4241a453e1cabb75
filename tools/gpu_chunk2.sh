#!/bin/bash
# Chunked updates, round 2: parity, then band / urgent-CTA / chunk sweeps.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_dag.py tests/test_gpu_xl.py tests/test_gpu_tuning.py -x -q --timeout=600 -p no:cacheprovider > gpurun_out/pytest_chunk2.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_chunk2.log
run() { timeout -s KILL 60 python tools/dag_bandsweep.py "$@"; }
{
for ch in 1 4 6 8; do for cfg in "cholesky 4000 250 50" "cholesky 4000 250 40" "lu 4000 250 40" "lu 4000 160 50" "lu 2000 200 40"; do TT_DAG_CHUNK=$ch run $cfg; done; done
for band in 3 6 9; do for u in 8 16 24; do for cfg in "cholesky 4000 250 40" "lu 4000 250 40"; do TT_DAG_BAND=$band TT_DAG_URGENT_CTAS=$u run $cfg; done; done; done
for m in "0,0" "750,250" "1500,100"; do for cfg in "cholesky 4000 250 40" "lu 4000 250 40"; do TT_DAG_MERGE=$m run $cfg; done; done
} > gpurun_out/chunk_sweep2.jsonl 2>&1
python3 - <<'PY'
import json
for l in open("gpurun_out/chunk_sweep2.jsonl"):
    try: r=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(r['kernel'], r['n'], r['by'], r['bx'], 'chunk', r['chunk'], 'band', r['band'], 'ucta', r['ucta'], 'merge', r['merge'], '%.3f ms %.2f TF %.1f%%' % (r['ms'], r['tflops'], 100*r['tflops']/37.05))
PY
