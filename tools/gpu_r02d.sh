#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_dag.py tests/test_gpu_xl.py tests/test_gpu_tuning.py -x -q --timeout=600 -p no:cacheprovider > gpurun_out/pytest_r02d.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_r02d.log
python tools/tune.py --kernel cholesky --size extralarge --evals 60 --seed 1 --devices 0 --trace > gpurun_out/tune_r02d.json 2>&1; tail -c 400 gpurun_out/tune_r02d.json | cut -c1-300
python tools/sweep.py --kernel cholesky --n 4000 --max-seconds 200 > gpurun_out/sweep_chol4000_r02d.jsonl 2>&1; tail -1 gpurun_out/sweep_chol4000_r02d.jsonl
python tools/sweep.py --kernel lu --n 4000 --max-seconds 200 > gpurun_out/sweep_lu4000_r02d.jsonl 2>&1; tail -1 gpurun_out/sweep_lu4000_r02d.jsonl
python tools/sweep.py --kernel lu --n 2000 --max-seconds 150 > gpurun_out/sweep_lu2000_r02d.jsonl 2>&1; tail -1 gpurun_out/sweep_lu2000_r02d.jsonl
