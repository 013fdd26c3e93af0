#!/bin/bash
mkdir -p gpurun_out/r2/san3
python tools/sanitize_run.py > gpurun_out/r2/san3/plain.log 2>&1; echo "plain rc=$?"; tail -14 gpurun_out/r2/san3/plain.log
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $CS --tool memcheck --leak-check no --print-limit 50 python tools/sanitize_run.py > gpurun_out/r2/san3/memcheck.log 2>&1; echo "memcheck rc=$?"; tail -3 gpurun_out/r2/san3/memcheck.log
timeout 1500 $CS --tool synccheck --print-limit 50 python tools/sanitize_run.py --quick > gpurun_out/r2/san3/synccheck.log 2>&1; echo "synccheck rc=$?"; tail -3 gpurun_out/r2/san3/synccheck.log
timeout 1800 $CS --tool racecheck --racecheck-report all --print-limit 50 python tools/sanitize_run.py --quick > gpurun_out/r2/san3/racecheck.log 2>&1; echo "racecheck rc=$?"; tail -3 gpurun_out/r2/san3/racecheck.log
