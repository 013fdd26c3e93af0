#!/bin/bash
mkdir -p gpurun_out/r2c
ncu --set full --clock-control none --import-source on -k regex:tree_conv -s 3 -c 1 -o gpurun_out/r2c/conv16 python tools/prof_conv.py --ncu > /dev/null 2>&1
ncu -i gpurun_out/r2c/conv16.ncu-rep --page details | grep -E "Duration|Executed Ipc|Issue Slots|Registers Per|Achieved Occ|Theoretical Occ|Executed Instructions  |DRAM Throughput|Block Limit"
ncu -i gpurun_out/r2c/conv16.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r2c/src16.csv 2>/dev/null
python tools/ncu_stalls.py gpurun_out/r2c/src16.csv stree_conv.cu 100 260 > gpurun_out/r2c/stalls16.txt; head -40 gpurun_out/r2c/stalls16.txt
