mkdir -p gpurun_out
timeout -s KILL 400 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
for cfg in "lu 2000 400,50" "lu 2000 125,64" "cholesky 4000 125,64" "lu 4000 250,64"; do
  set -- $cfg
  timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launch_$1_$2_$3.csv python tools/one_run.py --kernel $1 --dims $2 --cfg $3 --runs 2 > /dev/null 2>&1; echo "ncu $cfg rc=$?"
done
timeout -s KILL 150 python tools/sweep.py --kernel lu --n 2000 --min-bx 16 --max-seconds 60 > gpurun_out/sweep_lu2000.jsonl 2>&1; echo "sweep rc=$?"; tail -1 gpurun_out/sweep_lu2000.jsonl
timeout -s KILL 150 python tools/sweep.py --kernel cholesky --n 4000 --min-bx 32 --max-seconds 60 > gpurun_out/sweep_chol4000.jsonl 2>&1; echo "sweep rc=$?"; tail -1 gpurun_out/sweep_chol4000.jsonl
