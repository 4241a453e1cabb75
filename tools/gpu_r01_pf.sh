cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for pf in 0 1 2 3; do
  for cfg in "lu 2000 250 50" "cholesky 4000 250 50" "lu 4000 160 50"; do
    TT_DAG_PREFETCH=$pf timeout 120 python tools/dag_bandsweep.py $cfg
  done
done 2>&1 | grep -v Warn | tee gpurun_out/pf_sweep.jsonl
for u in 4 12 16; do for b in 2 3 4; do
  TT_DAG_URGENT_CTAS=$u TT_DAG_BAND=$b timeout 120 python tools/dag_bandsweep.py lu 2000 250 50
done; done 2>&1 | tee -a gpurun_out/pf_sweep.jsonl
TT_DAG_PREFETCH=2 timeout 200 python tools/dag_trace.py lu 2000 250 50 gpurun_out/tr_lu2000_pf.npz 2>&1 | tail -12
timeout 600 python -m pytest tests/test_gpu_dag.py -x -q 2>&1 | tail -2
