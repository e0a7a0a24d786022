#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; tail -2 gpurun_out/build.log
for kc in 4 8 16; do KC=$kc timeout 300 python tools/oz_perf.py 65536 1024 1 2>&1 | grep -E "engine=|chain|sched" | sed "s/^/KC=$kc /"; done 2>&1 | tee gpurun_out/kc_sweep.log
