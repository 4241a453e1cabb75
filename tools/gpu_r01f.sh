mkdir -p gpurun_out
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"dag_kernel" -s 1 -c 1 -o gpurun_out/prof_dag_lu2000 python tools/one_run.py --kernel lu --dims 2000 --cfg 400,50 --runs 2 > gpurun_out/ncu_dag.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_dag.log
