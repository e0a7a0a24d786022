#!/bin/bash
# usage: tools/gpu_tests.sh [pytest args...]   (runs on the GPU box via gpurun)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/build.log 2>&1; tail -3 gpurun_out/build.log
timeout 1500 python -m pytest tests -q -m gpu -p no:randomly "$@" > gpurun_out/pytest_gpu.log 2>&1; tail -15 gpurun_out/pytest_gpu.log
