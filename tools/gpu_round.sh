#!/bin/bash
# One gpurun call: tests, bench, ncu launch list, ncu --set full of the chain kernel.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -c 3000 gpurun_out/bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 1 --warmup 0 --no-e2e --no-cusolver --no-cpu > gpurun_out/bench_ncu.log 2>&1; tail -3 gpurun_out/bench_ncu.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chain -s 40 -c 2 -o gpurun_out/prof_chain -f \
   python tools/quick_perf.py 32768:1024 > gpurun_out/ncu_full.log 2>&1; tail -3 gpurun_out/ncu_full.log
