#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; tail -2 gpurun_out/build.log
timeout 240 python -m pytest tests/test_gpu_zz_multirank.py -q -k ozaki 2>&1 | grep -E "first timeout|passed|failed|Error" | head -4
timeout 300 python -m pytest tests/test_gpu_zz_multirank.py -q 2>&1 | grep -E "first timeout|passed|failed|Error" | head -4
