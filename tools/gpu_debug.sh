mkdir -p gpurun_out
export CUDA_LAUNCH_BLOCKING=1
TT_EAGER=1 timeout -s KILL 300 python tools/debug_variants.py > gpurun_out/debug_variants.log 2>&1; echo "debug rc=$?"
grep -v "OK$" gpurun_out/debug_variants.log | tail -30
TT_EAGER=1 timeout -s KILL 600 compute-sanitizer --tool memcheck --print-limit 100 python tools/debug_variants.py > gpurun_out/debug_sanitizer.log 2>&1; echo "sanitizer rc=$?"
grep -v "OK$" gpurun_out/debug_sanitizer.log | head -80
