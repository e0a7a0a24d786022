#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; tail -2 gpurun_out/build.log
for kc in 4 16; do KC=$kc timeout 300 python tools/oz_perf.py 65536 1024 1 2>&1 | grep -E "engine=|chain" | sed "s/^/KC=$kc /"; done 2>&1 | tee gpurun_out/kc_sweep.log
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:k_tc -c 1 -o gpurun_out/prof_tc_full -f \
   python bench.py --steps 1 --warmup 0 --no-e2e --no-cusolver --no-cpu --no-mxp --no-ooc --no-engine-compare > gpurun_out/ncu_tc_full.log 2>&1; tail -c 300 gpurun_out/ncu_tc_full.log
