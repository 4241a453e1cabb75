mkdir -p gpurun_out
timeout -s KILL 500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
timeout -s KILL 300 python tools/scaled_mm3.py --n 16384 --steps 2 --warmup 1 > gpurun_out/scaled16k.json 2>&1; echo "scaled16k rc=$?"; tail -2 gpurun_out/scaled16k.json
timeout -s KILL 400 python tools/scaled_mm3.py --n 32768 --steps 1 --warmup 1 > gpurun_out/scaled32k.json 2>&1; echo "scaled32k rc=$?"; tail -2 gpurun_out/scaled32k.json
timeout -s KILL 600 python tools/tune.py --kernel 3mm --size extralarge --evals 200 --trace > gpurun_out/tune_3mm_xl.json 2>&1; echo "tune3mm rc=$?"; tail -c 600 gpurun_out/tune_3mm_xl.json
timeout -s KILL 400 python tools/tune.py --kernel cholesky --size extralarge --evals 60 --trace > gpurun_out/tune_chol_xl.json 2>&1; echo "tunechol rc=$?"; tail -c 600 gpurun_out/tune_chol_xl.json
