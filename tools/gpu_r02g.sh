#!/bin/bash
# Round-2 state check: GPU tests, smoke, bench, XL knob sweep on the persistent kernel.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q --timeout=400 -p no:cacheprovider > gpurun_out/pytest_gpu_g.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu_g.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_g.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_g.log
timeout -s KILL 900 python bench.py > gpurun_out/bench_g.json 2> gpurun_out/bench_g.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench_g.json; echo; tail -3 gpurun_out/bench_g.err
for k in cholesky lu; do for bx in 32 40 50 80 100 125 160 200 250; do for by in 200 250 400 500 1000; do
  timeout -s KILL 60 python tools/dag_bandsweep.py $k 4000 $by $bx
done; done; done > gpurun_out/xl_sweep_g.jsonl 2>&1
python3 - <<'PY'
import json
rows=[]
for l in open("gpurun_out/xl_sweep_g.jsonl"):
    try: r = json.loads(l)
    except Exception: print(l[:200]); continue
    rows.append(r)
for r in sorted(rows, key=lambda r:(r["kernel"], r["ms"])):
    print(r["kernel"], r["n"], r["by"], r["bx"], "%.3f ms %.2f TF" % (r["ms"], r["tflops"]))
PY
