#!/bin/bash
# sharded outputs + symmetric memory (1 rank) + racecheck/memcheck of MSS + benches (default c4, force-heads c4)
mkdir -p gpurun_out/r2/san
timeout 900 python -m pytest -x -q --timeout 180 tests/test_sharded_gpu.py tests/test_mss_gpu.py tests/test_replay_gpu.py tests/test_pdl_gpu.py > gpurun_out/r2/pytest_s7.log 2>&1
tail -3 gpurun_out/r2/pytest_s7.log
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1200 $CS --tool racecheck --racecheck-report all --print-limit 200 python -m pytest -q -p no:cacheprovider tests/test_mss_gpu.py -k "random_trees and 1000" > gpurun_out/r2/san/racecheck_mss.log 2>&1; echo "racecheck mss rc=$?"; tail -2 gpurun_out/r2/san/racecheck_mss.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-next --no-cpu-baseline > gpurun_out/r2/bench7_c4.json 2> gpurun_out/r2/bench7_c4.err
timeout 600 python bench.py --steps 20 --warmup 5 --no-next --no-cpu-baseline --force-heads > gpurun_out/r2/bench7_c4_heads1.json 2> gpurun_out/r2/bench7_c4_heads1.err
for f in bench7_c4 bench7_c4_heads1; do python -c "import json; d=json.loads(open('gpurun_out/r2/$f.json').read().strip().splitlines()[-1]); k=d['roofline']['kernels']; print('$f', round(d['value']/1e6,2), d['parallelism'], {n: (round(v['us'],3) if 'us' in v else v) for n, v in k.items()}, 'e2e', round(d['e2e']['value']/1e6,2))"; done
tail -3 gpurun_out/r2/bench7_c4_heads1.err
