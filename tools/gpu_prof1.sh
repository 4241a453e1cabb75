mkdir -p gpurun_out
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"lu_panel|lu_trsm|dgemm_kernel" -s 40 -c 4 -o gpurun_out/prof_lu python tools/one_run.py --kernel lu --dims 2000 --cfg 400,50 --runs 1 > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_full.log
ls -la gpurun_out
