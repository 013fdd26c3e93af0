#!/bin/bash
# Round evidence on one GPU: full GPU test suite, smoke, bench lines (c4 default, c3, c2, --no-fuse, --force-heads,
# --impl reference), then the ncu launch lists / --set full captures (tools/profile_round.sh).
O=${O:-gpurun_out/ev}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/smi.txt
timeout 1200 python -m pytest tests -m gpu -q -rs > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for c in c3 c2; do timeout 300 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 300 python bench.py --no-fuse --no-next --no-cpu-baseline > $O/bench_nofuse.json 2> $O/bench_nofuse.err
timeout 300 python bench.py --force-heads --no-next --no-cpu-baseline > $O/bench_forceheads.json 2> $O/bench_forceheads.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
OUT=$O/prof timeout 1800 bash tools/profile_round.sh > $O/profile.log 2>&1
tail -3 $O/pytest_gpu.log; tail -1 $O/smoke.log
