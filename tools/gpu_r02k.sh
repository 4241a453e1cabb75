#!/bin/bash
# 3mm knob -> CTA region remap: parity + BO best-found over seeds.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_xl.py -m gpu -x -q -k "mm3 or 3mm or gemm" -p no:cacheprovider 2>&1 | tail -3
timeout -s KILL 1200 python tools/t1t8.py --kernel 3mm --size extralarge --evals 200 --workers 8 --seeds 1,2,3 --out gpurun_out/t1t8_3mm_xl_b.jsonl 2>&1 | tail -4
