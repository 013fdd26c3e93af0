#!/bin/bash
mkdir -p gpurun_out/r2k
O=gpurun_out/r2k
ncu --set full --clock-control none --import-source on -k regex:scan_tc128 -s 6 -c 1 -o $O/k2b_b16 \
    python tools/gpu/k2b_drive.py 16 128 > $O/ncu.log 2>&1
ncu -i $O/k2b_b16.ncu-rep --page source --csv --print-source cuda,sass > $O/src.csv 2>/dev/null
python tools/ncu_lines.py $O/src.csv 40 > $O/lines.txt; head -40 $O/lines.txt
ncu -i $O/k2b_b16.ncu-rep --page details > $O/details.txt; grep -E "Duration|Registers|Issue Slots|No Eligible|Active Warps|DRAM Through|Theoretical Occ" $O/details.txt
bash tools/gpu/r2_tr128.sh 2>&1 | head -60
