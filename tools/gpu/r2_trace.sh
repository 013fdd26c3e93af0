#!/bin/bash
mkdir -p gpurun_out/r2
timeout 300 python -m pytest -x -q tests/test_pdl_gpu.py > gpurun_out/r2/pytest_pdl.log 2>&1; tail -2 gpurun_out/r2/pytest_pdl.log
for f in 7 1; do timeout 120 python tools/trace_lat.py --config c3 --flags $f > gpurun_out/r2/tracelat_c3_f$f.txt 2>&1; done
timeout 120 python tools/trace_lat.py --config c3 --flags 7 --fused 0 > gpurun_out/r2/tracelat_c3_scan.txt 2>&1
timeout 120 python tools/trace_lat.py --config c2 --flags 7 > gpurun_out/r2/tracelat_c2_f7.txt 2>&1
