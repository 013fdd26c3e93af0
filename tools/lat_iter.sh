#!/bin/bash
# One GPU iteration on the small-batch kernel: build, GPU tests, c3/c2 bench lines, STREE_TRACE timelines (flags 31).
O=${O:-gpurun_out/lat}
mkdir -p $O
python -m paper_2505_14969_b200.build > $O/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for c in c3 c2; do timeout 300 python bench.py --config $c --no-next --no-cpu-baseline --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err; done
STREE_TRACE=1 python -m paper_2505_14969_b200.build > /dev/null 2>&1
timeout 120 python tools/trace_lat.py --config c3 --fused 1 --flags 31 --layers 16 > $O/trace_c3_fused.txt 2>&1
timeout 120 python tools/trace_lat.py --config c3 --fused 0 --flags 31 --layers 16 > $O/trace_c3_scan.txt 2>&1
python -m paper_2505_14969_b200.build --force > /dev/null 2>&1
tail -2 $O/pytest.log
for c in c3 c2; do python -c "
import json;d=json.load(open('$O/bench_$c.json'));r=d['roofline'];print('$c',round(d['value']/1e6,2),'M nodes/s',{k:round(v.get('us'),3) for k,v in r['kernels'].items()})"; done
