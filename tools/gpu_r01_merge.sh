cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TT_DAG_MERGE=700,100 timeout 600 python -m pytest tests/test_gpu_dag.py -x -q 2>&1 | tail -2
for m in 0,0 500,200 700,200 1000,200 1500,200 700,100 700,300 1000,100 1000,300; do
  for cfg in "lu 2000 250 50" "cholesky 4000 250 50" "lu 4000 160 50" "lu 2000 400 50" "cholesky 4000 500 50" "lu 2000 100 40"; do
    TT_DAG_MERGE=$m timeout 120 python tools/dag_bandsweep.py $cfg | sed "s/}/, \"merge\": \"$m\"}/"
  done
done 2>&1 | tee gpurun_out/merge_sweep2.jsonl
