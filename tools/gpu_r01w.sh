for cfg in "lu 2000 250 50" "lu 2000 200 40" "cholesky 4000 250 50" "lu 4000 160 50"; do
 for band in 2 3 4 6; do
  for uc in 8 16 32; do
   TT_DAG_BAND=$band TT_DAG_URGENT_CTAS=$uc timeout -s KILL 60 python tools/dag_bandsweep.py $cfg
  done
 done
done
