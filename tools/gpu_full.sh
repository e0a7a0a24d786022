#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/build.log 2>&1; tail -2 gpurun_out/build.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -I paper_2410_09819_b200/csrc -o tools/oz_test tools/oz_test.cu
timeout 120 ./tools/oz_test 8 2>&1 | tee gpurun_out/oz_test.log
timeout 300 python tools/oz_perf.py 65536 1024 1 2>&1 | grep -E "engine=|chain" | tee gpurun_out/oz_perf.log
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -6 gpurun_out/pytest_gpu.log
timeout 1500 python bench.py > gpurun_out/bench.log 2>&1; tail -c 300 gpurun_out/bench.log
