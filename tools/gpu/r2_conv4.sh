#!/bin/bash
mkdir -p gpurun_out/r2c
timeout 600 python -m pytest -x -q --timeout 300 tests/test_conv_gpu.py 2>&1 | tail -2
python tools/prof_conv.py 2>&1 | head -2
ncu --set full --clock-control none --import-source on -k regex:tree_conv -s 3 -c 1 -o gpurun_out/r2c/conv python tools/prof_conv.py --ncu > /dev/null 2>&1
ncu -i gpurun_out/r2c/conv.ncu-rep --page details | grep -E "Duration|Executed Ipc|Issue Slots|Registers Per|Achieved Occ|Executed Instructions  "
ncu -i gpurun_out/r2c/conv.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r2c/src.csv 2>/dev/null
python tools/ncu_stalls.py gpurun_out/r2c/src.csv stree_conv.cu 1 400 | head -30
