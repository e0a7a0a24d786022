#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -4 gpurun_out/pytest_gpu.log
NO_CUSOLVER=1 timeout 300 python tools/quick_perf.py 65536:1024 2>&1 | grep -E "TF/s probe|KC="
MXP=1e-5 NO_CUSOLVER=1 timeout 300 python tools/quick_perf.py 65536:1024 2>&1 | grep -E "TF/s probe|KC="
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
   python bench.py --steps 1 --warmup 0 --no-e2e --no-cusolver --no-cpu > gpurun_out/bench_ncu.log 2>&1; tail -c 600 gpurun_out/bench_ncu.log
