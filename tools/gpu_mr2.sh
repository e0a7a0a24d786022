#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; tail -2 gpurun_out/build.log
for i in 1 2 3 4; do timeout 600 python -m pytest tests/test_gpu_multirank.py -q -x 2>&1 | grep -E "first timeout|passed|failed" | head -3; done
timeout 600 python tools/mxp_perf.py 65536 2>&1 | tee gpurun_out/mxp_perf.log
