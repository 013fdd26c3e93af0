#!/bin/bash
# lat kernel v2: parity, bench c3/c2, trace
mkdir -p gpurun_out/r2
timeout 600 python -m pytest -x -q --timeout 120 tests/test_replay_gpu.py tests/test_parity_gpu.py tests/test_pdl_gpu.py > gpurun_out/r2/pytest_lat2.log 2>&1
tail -3 gpurun_out/r2/pytest_lat2.log
for c in c3 c2; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-next --no-cpu-baseline --no-e2e > gpurun_out/r2/bench2_$c.json 2> gpurun_out/r2/bench2_$c.err
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-next --no-cpu-baseline --no-e2e --no-fuse > gpurun_out/r2/bench2_${c}_nofuse.json 2>> gpurun_out/r2/bench2_$c.err
  python -c "import json; d=json.loads(open('gpurun_out/r2/bench2_$c.json').read().strip().splitlines()[-1]); print('$c', d['value'], d['ms_per_step'], d['roofline']['kernels'])"
  python -c "import json; d=json.loads(open('gpurun_out/r2/bench2_${c}_nofuse.json').read().strip().splitlines()[-1]); print('$c nofuse', d['value'], d['ms_per_step'], d['roofline']['kernels'])"
done
STREE_TRACE=1 python -c "from paper_2505_14969_b200 import build; build.build(force=True)" > /dev/null 2>&1
for f in 15 7; do timeout 120 python tools/trace_lat.py --config c3 --flags $f > gpurun_out/r2/tracelat2_c3_f$f.txt 2>&1; done
timeout 120 python tools/trace_lat.py --config c3 --flags 15 --fused 0 > gpurun_out/r2/tracelat2_c3_scan.txt 2>&1
head -1 gpurun_out/r2/tracelat2_*.txt
