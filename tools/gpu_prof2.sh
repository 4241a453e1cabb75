mkdir -p gpurun_out
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"panel_kernel|trsm_u_kernel" -s 20 -c 2 -o gpurun_out/prof_panel python tools/one_run.py --kernel lu --dims 2000 --cfg 400,50 --runs 1 > gpurun_out/ncu_full2.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_full2.log
