#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/build.log 2>&1; tail -2 gpurun_out/build.log
timeout 1500 python bench.py > gpurun_out/bench.log 2>&1; tail -c 300 gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; tail -c 400 gpurun_out/bench_ref.log
