#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dmma_bench tools/dmma_bench.cu > /dev/null 2>&1
timeout 300 /tmp/dmma_bench 2>&1 | tee gpurun_out/dmma_bench.log
timeout 900 python bench.py --no-e2e > gpurun_out/bench.log 2>&1; tail -c 2500 gpurun_out/bench.log
