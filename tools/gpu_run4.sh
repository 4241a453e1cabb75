mkdir -p gpurun_out
timeout -s KILL 120 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
timeout -s KILL 400 python -m pytest tests -q -m gpu -x --durations=5 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -12 gpurun_out/pytest_gpu.log
timeout -s KILL 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -2 gpurun_out/bench.log | cut -c1-1500
timeout -s KILL 150 python tools/sweep.py --kernel lu --n 2000 --min-bx 16 --max-seconds 100 > gpurun_out/sweep_lu2000.jsonl 2>&1; echo "sweep rc=$?"; tail -1 gpurun_out/sweep_lu2000.jsonl
timeout -s KILL 150 python tools/sweep.py --kernel cholesky --n 4000 --min-bx 32 --max-seconds 100 > gpurun_out/sweep_chol4000.jsonl 2>&1; echo "sweep rc=$?"; tail -1 gpurun_out/sweep_chol4000.jsonl
timeout -s KILL 150 python tools/sweep.py --kernel lu --n 4000 --min-bx 32 --max-seconds 100 > gpurun_out/sweep_lu4000.jsonl 2>&1; echo "sweep rc=$?"; tail -1 gpurun_out/sweep_lu4000.jsonl
