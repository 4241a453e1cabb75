mkdir -p gpurun_out
timeout -s KILL 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -3 gpurun_out/bench.log
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lu_launches.csv python tools/one_run.py --kernel lu --dims 2000 --cfg 400,50 --runs 2 > gpurun_out/ncu_lu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_lu.log
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lu2000_launches.csv python tools/one_run.py --kernel lu --dims 2000 --cfg 80,2000 --runs 2 > gpurun_out/ncu_lu2.log 2>&1; echo "ncu2 rc=$?"
timeout -s KILL 400 python -m pytest tests -q -m gpu --durations=5 -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
