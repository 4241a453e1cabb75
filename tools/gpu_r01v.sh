mkdir -p gpurun_out
timeout -s KILL 200 python tools/sweep.py --kernel lu --n 2000 --min-bx 8 --max-seconds 150 > gpurun_out/sweep_lu2000.jsonl 2> gpurun_out/sweep_lu2000.err; echo "sweep lu rc=$?"
python3 -c "
import json
rows=[json.loads(l) for l in open('gpurun_out/sweep_lu2000.jsonl') if l.strip().startswith('{')]
rows=[r for r in rows if 'gflops' in r]
rows.sort(key=lambda r:-r['gflops'])
for r in rows[:12]: print(r)
print(len(rows),'configs')
"
timeout -s KILL 200 python tools/sweep3mm.py --size large --samples 600 --max-seconds 120 > gpurun_out/sweep3mm_large.jsonl 2>&1; echo "sweep3mm rc=$?"; cat gpurun_out/sweep3mm_large.jsonl
timeout -s KILL 300 python tools/tune.py --kernel cholesky --size extralarge --evals 60 > gpurun_out/tune_chol_xl.json 2>&1; echo "tune chol rc=$?"; head -c 600 gpurun_out/tune_chol_xl.json
