mkdir -p gpurun_out
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"panel_kernel" -s 10 -c 1 -o gpurun_out/prof_panel2 python tools/one_run.py --kernel lu --dims 2000 --cfg 400,50 --runs 1 > gpurun_out/ncu_full3.log 2>&1; echo "ncu rc=$?"
