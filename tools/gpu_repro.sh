#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for rep in 1 2; do
timeout -s KILL 300 python tools/sweep.py --kernel lu --n 2000 --min-bx 8 --max-seconds 200 > gpurun_out/rep_lu2000_$rep.jsonl 2>&1; grep -c '"kernel"' gpurun_out/rep_lu2000_$rep.jsonl; grep -i "watchdog" gpurun_out/rep_lu2000_$rep.jsonl | tail -1
timeout -s KILL 400 python tools/sweep.py --kernel lu --n 4000 --min-bx 16 --max-seconds 300 > gpurun_out/rep_lu4000_$rep.jsonl 2>&1; grep -c '"kernel"' gpurun_out/rep_lu4000_$rep.jsonl; grep -i "watchdog" gpurun_out/rep_lu4000_$rep.jsonl | tail -1
done
