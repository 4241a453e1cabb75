mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout -s KILL 600 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
timeout -s KILL 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout -s KILL 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_lu.csv python tools/one_run.py --kernel lu --dims 2000 --cfg 400,50 --runs 2 > gpurun_out/ncu_launch.log 2>&1; echo "ncu launch rc=$?"
python tools/launch_summary.py gpurun_out/launches_lu.csv
timeout -s KILL 400 ncu --set full --clock-control none --import-source on -k regex:"dgemm" -s 20 -c 1 -o gpurun_out/prof_lu_dgemm python tools/one_run.py --kernel lu --dims 2000 --cfg 400,50 --runs 1 > gpurun_out/ncu_full1.log 2>&1; echo "ncu full dgemm rc=$?"
timeout -s KILL 400 ncu --set full --clock-control none --import-source on -k regex:"panel_kernel" -s 10 -c 1 -o gpurun_out/prof_lu_panel python tools/one_run.py --kernel lu --dims 2000 --cfg 400,50 --runs 1 > gpurun_out/ncu_full2.log 2>&1; echo "ncu full panel rc=$?"
