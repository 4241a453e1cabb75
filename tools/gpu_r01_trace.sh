cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 200 python tools/dag_trace.py lu 2000 250 50 gpurun_out/tr_lu2000.npz 2>&1 | tail -20
timeout 200 python tools/dag_trace.py cholesky 4000 250 50 gpurun_out/tr_ch4000.npz 2>&1 | tail -20
