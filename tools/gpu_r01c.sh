mkdir -p gpurun_out
timeout -s KILL 300 python tools/dag_check.py > gpurun_out/dag_check.log 2>&1; echo "dag_check rc=$?"; cat gpurun_out/dag_check.log | tail -30
timeout -s KILL 600 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
