#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
timeout -s KILL 300 python tools/sweep3mm.py --size extralarge --samples 300 --max-seconds 100 2>&1 | tail -4
timeout -s KILL 300 python tools/sweep3mm.py --size large --samples 300 --max-seconds 60 2>&1 | tail -4
timeout -s KILL 1200 python tools/t1t8.py --kernel 3mm --size extralarge --evals 200 --workers 8 --seeds 1,2,3 --out gpurun_out/t1t8_3mm_xl_d.jsonl 2>&1 | tail -4
