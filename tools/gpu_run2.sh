mkdir -p gpurun_out
timeout -s KILL 120 python tools/debug_gemm.py > gpurun_out/debug_gemm.log 2>&1; echo "dbg rc=$?"
cat gpurun_out/debug_gemm.log | tail -40
timeout -s KILL 120 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
timeout -s KILL 200 python tools/sweep.py --kernel lu --n 2000 --min-bx 16 --max-seconds 100 > gpurun_out/sweep_lu2000.jsonl 2>&1; echo "sweep rc=$?"
tail -2 gpurun_out/sweep_lu2000.jsonl
timeout -s KILL 400 python -m pytest tests -q -m gpu --durations=15 -k "not gemm_tile" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/pytest_gpu.log
