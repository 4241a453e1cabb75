cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dag.py tests/test_gpu_kernels.py -x -q 2>&1 | tail -2
timeout 200 python tools/dag_trace.py lu 2000 250 50 gpurun_out/tr_lu2000_m.npz 2>&1 | tail -12
timeout 200 python tools/dag_trace.py cholesky 4000 250 50 gpurun_out/tr_ch4000_m.npz 2>&1 | tail -12
