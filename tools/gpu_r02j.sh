#!/bin/bash
# C++ drop-in on the GPU, T1/T8 virtual-clock time-to-best (3mm XL, Cholesky XL), urgent-chain trace.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_dropin.py -q -s -p no:cacheprovider 2>&1 | tail -20
timeout -s KILL 1200 python tools/t1t8.py --kernel 3mm --size extralarge --evals 200 --workers 8 --seeds 1,2,3 --out gpurun_out/t1t8_3mm_xl.jsonl 2>&1 | tail -5
timeout -s KILL 900 python tools/t1t8.py --kernel cholesky --size extralarge --evals 60 --workers 8 --seeds 1,2,3 --out gpurun_out/t1t8_chol_xl.jsonl 2>&1 | tail -5
timeout -s KILL 200 python tools/dag_trace.py cholesky 4000 1000 160 gpurun_out/tr_chol_1000_160.npz 2>&1 | tail -3
