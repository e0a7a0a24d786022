#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; tail -2 gpurun_out/build.log
timeout 900 python -m pytest tests/test_gpu_mxp.py tests/test_gpu_ozaki.py tests/test_gpu_loglik.py -q 2>&1 | tail -2
timeout 1200 python bench.py --no-e2e --no-cusolver --no-cpu --no-ooc --no-engine-compare > gpurun_out/bench_img4.log 2>&1; tail -c 200 gpurun_out/bench_img4.log
