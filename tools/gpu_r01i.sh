mkdir -p gpurun_out
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:bench -c 8 -o gpurun_out/prof_diag_bench ./tools/microbench/diag_bench > gpurun_out/ncu_diag.log 2>&1; echo rc=$?; tail -3 gpurun_out/ncu_diag.log
