#!/bin/bash
mkdir -p gpurun_out/r2/san
timeout 900 python -m pytest -x -q --timeout 180 tests/test_replay_gpu.py tests/test_parity_gpu.py tests/test_pdl_gpu.py tests/test_conv_gpu.py > gpurun_out/r2/pytest_s11.log 2>&1; tail -2 gpurun_out/r2/pytest_s11.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-next --no-cpu-baseline --no-e2e > gpurun_out/r2/bench11.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/r2/bench11.json').read().strip().splitlines()[-1]); k=d['roofline']['kernels']['stree_replay_scan']; print('c4', round(d['value']/1e6,2), round(k['us'],3), round(k['frac'],4), 'iso', round(k['isolated_call_us'],2))"
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 2400 $CS --tool racecheck --racecheck-report all --print-limit 2000 python tools/sanitize_run.py > gpurun_out/r2/san/racecheck_final.log 2>&1; echo "racecheck rc=$?"; tail -2 gpurun_out/r2/san/racecheck_final.log
timeout 1500 $CS --tool memcheck --leak-check no --print-limit 50 python tools/sanitize_run.py > gpurun_out/r2/san/memcheck_final.log 2>&1; echo "memcheck rc=$?"; tail -1 gpurun_out/r2/san/memcheck_final.log
timeout 1500 $CS --tool synccheck --print-limit 50 python tools/sanitize_run.py > gpurun_out/r2/san/synccheck_final.log 2>&1; echo "synccheck rc=$?"; tail -1 gpurun_out/r2/san/synccheck_final.log
