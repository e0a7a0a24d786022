#!/bin/bash
# One gpurun call: build, GPU tests, default bench, ncu launch list, ncu --set full of k_sched at the bench config.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/build.log 2>&1; tail -2 gpurun_out/build.log
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; tail -4 gpurun_out/pytest_gpu.log
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1; tail -c 400 gpurun_out/bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
   python bench.py --steps 1 --warmup 0 --no-e2e --no-cusolver --no-cpu --no-mxp --no-ooc > gpurun_out/bench_ncu.log 2>&1; tail -c 300 gpurun_out/bench_ncu.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_sched -c 1 -o gpurun_out/prof_sched_full -f \
   python bench.py --steps 1 --warmup 0 --no-e2e --no-cusolver --no-cpu --no-mxp --no-ooc > gpurun_out/ncu_full.log 2>&1; tail -c 300 gpurun_out/ncu_full.log
