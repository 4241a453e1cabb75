set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "batch or dag or lu_contracts" 2>&1 | tail -5
timeout 300 python bench.py > gpurun_out/bench_batch.json 2> gpurun_out/bench_batch.err; tail -3 gpurun_out/bench_batch.err
cat gpurun_out/bench_batch.json | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['e2e'], d['parity'])"
