mkdir -p gpurun_out
for c in "lu 2000 400 50" "cholesky 4000 500 50"; do
  set -- $c
  timeout -s KILL 120 python tools/dag_trace.py $c gpurun_out/trace_$1_$2_$3_$4.npz 2>&1 | grep -E "walker per|span"
done
