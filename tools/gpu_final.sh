#!/bin/bash
# round-end evidence (run under gpurun): smoke, the full default bench line, and the ncu launch
# list of the C2 leg (kernels serialized: its per-launch times are cold-cache)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/build.log 2>&1; tail -2 gpurun_out/build.log
timeout 1500 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; tail -c 300 gpurun_out/bench_full.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cusolver --no-cpu --no-mxp --no-ooc --no-engine-compare --no-kl \
    > gpurun_out/launches_c2.out 2>&1; echo launches rc=$?
