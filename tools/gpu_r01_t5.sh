cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dag.py tests/test_gpu_kernels.py -x -q 2>&1 | tail -2
for cfg in "lu 2000 250 50" "cholesky 4000 250 50" "lu 4000 160 50" "lu 2000 400 50" "lu 2000 100 40"; do
  timeout 120 python tools/dag_bandsweep.py $cfg
done 2>&1 | tee gpurun_out/t5_sweep.jsonl
timeout 200 python tools/dag_trace.py lu 2000 250 50 gpurun_out/tr_lu2000_v.npz 2>&1 | tail -12
