mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > gpurun_out/smi_before.txt
timeout -s KILL 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout -s KILL 400 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"; tail -c 1200 gpurun_out/bench_ref.json
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_lu_dag.csv python tools/one_run.py --kernel lu --dims 2000 --cfg 400,50 --runs 2 > gpurun_out/ncu_launch.log 2>&1; echo "ncu launch rc=$?"
timeout -s KILL 400 ncu --set full --clock-control none --import-source on -k regex:"dag_kernel" -s 1 -c 1 -o gpurun_out/prof_dag_lu2000_v6 python tools/one_run.py --kernel lu --dims 2000 --cfg 400,50 --runs 2 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
