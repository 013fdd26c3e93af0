#!/bin/bash
mkdir -p gpurun_out/r2
timeout 900 python -m pytest -x -q --timeout 180 tests/test_scan_tc128_gpu.py tests/test_parity_gpu.py > gpurun_out/r2/pytest_k2b.log 2>&1; tail -2 gpurun_out/r2/pytest_k2b.log
timeout 600 python tools/sweep_c5.py > gpurun_out/r2/sweep_c5_k2b.txt 2>&1; tail -25 gpurun_out/r2/sweep_c5_k2b.txt
