#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; tail -2 gpurun_out/build.log
timeout 900 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; tail -12 gpurun_out/bench.err; tail -c 300 gpurun_out/bench.log
