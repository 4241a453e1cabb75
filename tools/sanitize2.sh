#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
CS=/usr/local/cuda/bin/compute-sanitizer
timeout -s KILL 900 $CS --tool memcheck --print-limit 5 python tools/repro_run.py lu 4000 4000,40 1000,40 2>&1 | grep -E "ok|FAIL|ERROR|Invalid|of size|at 0x" | head -12
timeout -s KILL 900 $CS --tool memcheck --print-limit 5 python tools/repro_run.py cholesky 4000 1000,40 1000,160 2>&1 | grep -E "ok|FAIL|ERROR|Invalid|of size|at 0x" | head -12
timeout -s KILL 900 $CS --tool memcheck --print-limit 5 python tools/repro_run.py lu 2000 400,50 40,40 2000,2000 125,125 200,16 1000,8 2>&1 | grep -E "ok|FAIL|ERROR|Invalid|of size|at 0x" | head -12
timeout -s KILL 900 $CS --tool memcheck --print-limit 5 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k "mm3 or gemm" -p no:cacheprovider 2>&1 | grep -E "passed|failed|ERROR|Invalid|of size" | head -12
