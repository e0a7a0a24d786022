#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; tail -2 gpurun_out/build.log
timeout 900 python -m pytest tests/test_gpu_ozaki.py -q -x 2>&1 | grep -E "first timeout|passed|failed|Error" | head -20
timeout 300 python tools/oz_perf.py 65536 1024 1 2>&1 | grep -E "engine=|chain"
timeout 1500 python bench.py > gpurun_out/bench.log 2>&1; tail -c 600 gpurun_out/bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
   python bench.py --steps 1 --warmup 0 --no-e2e --no-cusolver --no-cpu --no-mxp --no-ooc --no-engine-compare > gpurun_out/bench_ncu.log 2>&1; tail -c 300 gpurun_out/bench_ncu.log
