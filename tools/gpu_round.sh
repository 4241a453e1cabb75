#!/bin/bash
# Round measurement on one B200 (run through gpurun from the repo root):
# GPU tests, smoke, both bench arms, the ncu launch list of the bench command
# and one ncu --set full capture of the headline kernel.  Outputs -> gpurun_out/.
# Usage: bash tools/gpu_round.sh <tag>
TAG=${1:-r01}
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests -m gpu -x -q --timeout=300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout -s KILL 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; tail -c 600 gpurun_out/bench_$TAG.json; echo; tail -2 gpurun_out/bench_$TAG.err
timeout -s KILL 600 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"; tail -c 400 gpurun_out/bench_ref_$TAG.json; echo
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu launch rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"dag_kernel" -s 1 -c 1 -o gpurun_out/prof_dag_lu2000_$TAG python tools/one_run.py --kernel lu --dims 2000 --cfg 200,40 --runs 2 > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
