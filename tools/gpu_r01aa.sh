for cfg in "lu 2000 250 50" "lu 2000 200 40" "lu 2000 400 50" "cholesky 4000 250 50" "cholesky 4000 500 50" "lu 4000 160 50" "lu 4000 200 40"; do
  timeout -s KILL 60 python tools/dag_bandsweep.py $cfg
done
