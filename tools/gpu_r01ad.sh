timeout -s KILL 300 python tools/dag_check.py 2>&1 | grep -v "dag=False"
for c in "lu 2000 250 50" "cholesky 4000 250 50"; do
  timeout -s KILL 120 python tools/dag_trace.py $c 2>&1 | grep -E "walker|span|TRSM|GEMM  "
done
timeout -s KILL 600 python -m pytest tests/test_gpu_dag.py tests/test_gpu_kernels.py -q -m gpu -x 2>&1 | tail -3
