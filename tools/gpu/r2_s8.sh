#!/bin/bash
mkdir -p gpurun_out/r2
timeout 600 python -m pytest -x -q --timeout 120 tests/test_conv_gpu.py > gpurun_out/r2/pytest_conv.log 2>&1; tail -3 gpurun_out/r2/pytest_conv.log
timeout 300 python -c "
import json, torch, bench_next
from bench import load_peaks
hbm, bf, _ = load_peaks()
r = bench_next.measure(torch.device('cuda', 0), hbm, bf)
print(json.dumps({k: v for k, v in r.items() if k in ('tree_conv', 'conv_commit')}))
" > gpurun_out/r2/next_conv.json 2> gpurun_out/r2/next_conv.err; cat gpurun_out/r2/next_conv.json; tail -2 gpurun_out/r2/next_conv.err
