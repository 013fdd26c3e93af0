#!/bin/bash
# racecheck after the K2b ancestor-jumping fix: every kernel family, hazards summarised by source line
mkdir -p gpurun_out/r2/san
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 2400 $CS --tool racecheck --racecheck-report all --print-limit 20000 python tools/sanitize_run.py > gpurun_out/r2/san/racecheck_full.log 2>&1; echo "racecheck rc=$?"
tail -3 gpurun_out/r2/san/racecheck_full.log
python tools/race_summary.py gpurun_out/r2/san/racecheck_full.log > gpurun_out/r2/san/racecheck_summary.txt; cat gpurun_out/r2/san/racecheck_summary.txt | tail -25
gzip -f gpurun_out/r2/san/racecheck_full.log
