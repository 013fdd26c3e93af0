#!/bin/bash
mkdir -p gpurun_out/r2 gpurun_out/r2/san
timeout 900 python -m pytest -x -q --timeout 180 tests/test_opts_gpu.py tests/test_conv_gpu.py > gpurun_out/r2/pytest_s10.log 2>&1; tail -15 gpurun_out/r2/pytest_s10.log
python tools/prof_conv.py | head -1
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 2400 $CS --tool racecheck --racecheck-report all --print-limit 2000 python tools/sanitize_run.py > gpurun_out/r2/san/racecheck_final.log 2>&1; echo "racecheck rc=$?"; tail -2 gpurun_out/r2/san/racecheck_final.log
