mkdir -p gpurun_out
timeout -s KILL 400 ncu --set full --clock-control none --import-source on -k regex:"dgemm_kernel" -s 3 -c 3 -o gpurun_out/prof_3mm_xl python tools/one_run.py --kernel 3mm --dims 1600,1800,2000,2200,2400 --cfg 64,125,125,120,64,120 --runs 2 > gpurun_out/ncu_3mm.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_3mm.log
