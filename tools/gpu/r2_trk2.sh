#!/bin/bash
mkdir -p gpurun_out/r2
STREE_TRACE=1 python -c "from paper_2505_14969_b200 import build; build.build(force=True)" > /dev/null 2>&1
timeout 120 python tools/trace_stack.py > gpurun_out/r2/trace_stack_c4.txt 2>&1; cat gpurun_out/r2/trace_stack_c4.txt
