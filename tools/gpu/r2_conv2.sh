#!/bin/bash
mkdir -p gpurun_out/r2
ncu --set full --clock-control none --import-source on -k regex:tree_conv -s 6 -c 1 -o gpurun_out/r2/ncu_conv_pipe python tools/prof_conv.py --ncu --layers 4 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:tree_conv -s 14 -c 1 -o gpurun_out/r2/ncu_conv_old python tools/prof_conv.py --ncu --layers 4 > /dev/null 2>&1
ls gpurun_out/r2/ncu_conv_*
