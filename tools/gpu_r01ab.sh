for c in "lu 2000 250 50" "cholesky 4000 250 50"; do
  timeout -s KILL 120 python tools/dag_trace.py $c 2>&1 | grep -E "walker|span"
done
