mkdir -p gpurun_out
for cfg in "lu 2000 400,50" "lu 2000 400,2000" "cholesky 4000 125,160" "lu 4000 500,32"; do
  set -- $cfg
  timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launch_$1_$2_$3.csv python tools/one_run.py --kernel $1 --dims $2 --cfg $3 --runs 2 > /dev/null 2>&1; echo "ncu $cfg rc=$?"
done
