#!/bin/bash
# Round-2 state check on one B200: GPU tests, smoke, bench (both arms), ncu launch
# list + one --set full capture of the headline kernel (Cholesky XL), T1/T8 replay.
TAG=${1:-r02a}
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q --timeout=600 -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_$TAG.log
timeout -s KILL 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench_$TAG.json; echo; tail -3 gpurun_out/bench_$TAG.err
timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"; tail -c 600 gpurun_out/bench_ref_$TAG.json; echo
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-extra --no-cpu-baseline --no-tuning > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu launch rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"dag_kernel" -s 1 -c 1 -o gpurun_out/prof_chol4000_$TAG python tools/one_run.py --kernel cholesky --dims 4000 --cfg 250,40 --runs 2 > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
timeout -s KILL 900 python tools/t1t8.py --kernel 3mm --size extralarge --evals 200 --workers 8 --seeds 1,2,3 --out gpurun_out/t1t8_3mm_$TAG.jsonl > gpurun_out/t1t8_$TAG.log 2>&1; echo "t1t8 rc=$?"; tail -2 gpurun_out/t1t8_$TAG.log
