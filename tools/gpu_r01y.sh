mkdir -p gpurun_out
timeout -s KILL 240 python tools/sweep3mm.py --size extralarge --samples 800 --max-seconds 180 > gpurun_out/sweep3mm_xl.jsonl 2>&1; echo "sweep3mm xl rc=$?"; cat gpurun_out/sweep3mm_xl.jsonl
timeout -s KILL 400 python tools/tune.py --kernel 3mm --size extralarge --evals 200 > gpurun_out/tune_3mm_xl.json 2>&1; echo "tune 3mm rc=$?"; head -c 500 gpurun_out/tune_3mm_xl.json
timeout -s KILL 300 python tools/tune.py --kernel lu --size large --evals 60 > gpurun_out/tune_lu_l.json 2>&1; echo "tune lu rc=$?"; head -c 500 gpurun_out/tune_lu_l.json
