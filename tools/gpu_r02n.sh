#!/bin/bash
# Knob sweeps (current kernels), BO runs for the bench's tuned configs, ncu traffic captures.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 300 python tools/sweep.py --kernel lu --n 2000 --min-bx 8 --max-seconds 200 > gpurun_out/sweep_lu2000_r02.jsonl 2>&1; tail -1 gpurun_out/sweep_lu2000_r02.jsonl
timeout -s KILL 400 python tools/sweep.py --kernel cholesky --n 4000 --min-bx 16 --max-seconds 300 > gpurun_out/sweep_chol4000_r02.jsonl 2>&1; tail -1 gpurun_out/sweep_chol4000_r02.jsonl
timeout -s KILL 400 python tools/sweep.py --kernel lu --n 4000 --min-bx 16 --max-seconds 300 > gpurun_out/sweep_lu4000_r02.jsonl 2>&1; tail -1 gpurun_out/sweep_lu4000_r02.jsonl
timeout -s KILL 900 python tools/t1t8.py --kernel cholesky --size extralarge --evals 60 --workers 8 --seeds 1,2,3 --out gpurun_out/t1t8_chol_xl_r02b.jsonl 2>&1 | tail -1
