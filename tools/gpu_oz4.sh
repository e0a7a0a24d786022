#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; tail -2 gpurun_out/build.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -I paper_2410_09819_b200/csrc -o tools/oz_test tools/oz_test.cu
timeout 120 ./tools/oz_test 8 2>&1 | tee gpurun_out/oz_test.log
timeout 120 ./tools/oz_test 7 2>&1 | tee -a gpurun_out/oz_test.log
timeout 900 python -m pytest tests/test_gpu_ozaki.py -q -x 2>&1 | grep -E "first timeout|passed|failed|Error" | head -20
timeout 600 python tools/oz_perf.py 65536 1024 1 2>&1 | tee gpurun_out/oz_perf.log
S=7 timeout 600 python tools/oz_perf.py 65536 1024 1 2>&1 | tee -a gpurun_out/oz_perf.log
