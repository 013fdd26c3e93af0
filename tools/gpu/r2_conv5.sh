#!/bin/bash
timeout 600 python -m pytest -x -q --timeout 300 tests/test_conv_gpu.py 2>&1 | tail -2
python tools/prof_conv.py 2>&1 | head -1
