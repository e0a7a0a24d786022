#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; tail -2 gpurun_out/build.log
for i in 1 2; do timeout 600 python -m pytest tests/test_gpu_zz_multirank.py -q 2>&1 | grep -E "first timeout|passed|failed|Error" | head -4; done
timeout 900 python -m pytest tests/test_gpu_ozaki.py -q 2>&1 | tail -1
