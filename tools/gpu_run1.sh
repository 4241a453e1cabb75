set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout -s KILL 120 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
tail -5 gpurun_out/smoke.log
timeout -s KILL 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu.log
timeout -s KILL 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -5 gpurun_out/bench.log
timeout -s KILL 200 python tools/sweep.py --kernel lu --n 2000 --max-seconds 150 > gpurun_out/sweep_lu2000.jsonl 2>&1; echo "sweep rc=$?"
tail -3 gpurun_out/sweep_lu2000.jsonl
