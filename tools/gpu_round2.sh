#!/bin/bash
# Round-2 measurement: smoke, both bench arms, ncu launch list of the bench command,
# ncu --set full of the headline kernel (Cholesky XL) and the 3mm XL kernels.
TAG=${1:-r02a}
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout -s KILL 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_$TAG.err
timeout -s KILL 600 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"; tail -c 300 gpurun_out/bench_ref_$TAG.json; echo
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-extra --no-cpu-baseline --no-tuning > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu launch rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"dag_kernel" -s 1 -c 1 -o gpurun_out/prof_chol_xl_$TAG python tools/one_run.py --kernel cholesky --dims 4000 --cfg 1000,40 --runs 2 > gpurun_out/ncu_full_chol_$TAG.log 2>&1; echo "ncu chol rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"dag_kernel" -s 1 -c 1 -o gpurun_out/prof_lu2000_$TAG python tools/one_run.py --kernel lu --dims 2000 --cfg 400,40 --runs 2 > gpurun_out/ncu_full_lu_$TAG.log 2>&1; echo "ncu lu rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"dgemm" -s 3 -c 3 -o gpurun_out/prof_3mm_xl_$TAG python tools/one_run.py --kernel 3mm --dims 1600,1800,2000,2200,2400 --cfg 2,1000,1000,4,1,2 --runs 2 > gpurun_out/ncu_full_3mm_$TAG.log 2>&1; echo "ncu 3mm rc=$?"
