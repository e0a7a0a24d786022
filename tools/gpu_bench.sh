#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; tail -2 gpurun_out/build.log
timeout 1500 python bench.py > gpurun_out/bench.log 2>&1; tail -c 600 gpurun_out/bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
   python bench.py --steps 1 --warmup 0 --no-e2e --no-cusolver --no-cpu --no-mxp --no-ooc --no-engine-compare > gpurun_out/bench_ncu.log 2>&1; tail -c 300 gpurun_out/bench_ncu.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_tc -c 1 -o gpurun_out/prof_tc_full -f \
   python bench.py --steps 1 --warmup 0 --no-e2e --no-cusolver --no-cpu --no-mxp --no-ooc --no-engine-compare > gpurun_out/ncu_tc_full.log 2>&1; tail -c 300 gpurun_out/ncu_tc_full.log
