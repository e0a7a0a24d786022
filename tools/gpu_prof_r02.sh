#!/bin/bash
# ncu evidence for round 2 (run under gpurun): launch list of the bench command, full captures
# of k_tc at C2 (Ozaki) and of k_tc on a native-engine MxP map.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-ooc --no-mxp --no-kl --no-cpu --no-cusolver --no-engine-compare \
    > gpurun_out/launches_r02.out 2>&1; echo launches rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tc -c 1 -o gpurun_out/k_tc_c2_r02 \
    python tools/oz_perf.py 65536 1024 1 > gpurun_out/k_tc_c2_r02.out 2>&1; echo k_tc rc=$?
DBG=0 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tc -c 1 -o gpurun_out/k_tc_native_r02 \
    python tools/mxp_perf.py 32768 1e-5 3 > gpurun_out/k_tc_native_r02.out 2>&1; echo native rc=$?
ls -la gpurun_out/*.ncu-rep
