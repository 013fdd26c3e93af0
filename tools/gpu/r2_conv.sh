#!/bin/bash
mkdir -p gpurun_out/r2
python tools/prof_conv.py
ncu --set full --clock-control none --import-source on -k regex:tree_conv -s 6 -c 2 -o gpurun_out/r2/ncu_conv python tools/prof_conv.py --ncu --layers 4 > gpurun_out/r2/ncu_conv.log 2>&1
tail -2 gpurun_out/r2/ncu_conv.log
