mkdir -p gpurun_out
timeout -s KILL 300 python tools/dag_check.py > gpurun_out/dag_check.log 2>&1; echo "dag_check rc=$?"; cat gpurun_out/dag_check.log | grep -v "dag=False"
for c in "lu 2000 400 50" "lu 2000 200 40" "cholesky 4000 500 50"; do
  set -- $c
  timeout -s KILL 120 python tools/dag_trace.py $c gpurun_out/trace_$1_$2_$3_$4.npz 2>&1 | tail -11
done
timeout -s KILL 600 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
