#!/bin/bash
# compute-sanitizer memcheck over small persistent-schedule and 3mm runs.
cd "${GRAFT_REPO_ROOT:-.}"
CS=/usr/local/cuda/bin/compute-sanitizer
timeout -s KILL 600 $CS --tool memcheck --print-limit 5 python tools/repro_run.py lu 400 100,40 400,40 200,50 80,16 400,8 2>&1 | grep -E "ok|FAIL|ERROR|Invalid|of size|at 0x|ERROR SUMMARY" | head -20
timeout -s KILL 600 $CS --tool memcheck --print-limit 5 python tools/repro_run.py cholesky 400 100,40 400,40 200,50 80,16 400,8 2>&1 | grep -E "ok|FAIL|ERROR|Invalid|of size|at 0x|ERROR SUMMARY" | head -20
timeout -s KILL 600 $CS --tool memcheck --print-limit 5 python tools/repro_run.py lu 1000 1000,40 250,40 2>&1 | grep -E "ok|FAIL|ERROR|Invalid|of size|at 0x|ERROR SUMMARY" | head -20
timeout -s KILL 600 $CS --tool memcheck --print-limit 5 python tools/repro_run.py cholesky 1000 1000,40 250,40 2>&1 | grep -E "ok|FAIL|ERROR|Invalid|of size|at 0x|ERROR SUMMARY" | head -20
