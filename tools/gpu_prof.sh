#!/bin/bash
# ncu --set full of k_tc at C2 (Ozaki) and on a native-engine MxP map (run under gpurun)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
REPS=2 python tools/perf_run.py c2 65536 1024; REPS=2 python tools/perf_run.py mxp 65536 1e-5
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tc -c 1 -f -o gpurun_out/k_tc_c2 \
    python tools/perf_run.py c2 65536 1024 > gpurun_out/k_tc_c2.out 2>&1; echo k_tc rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tc -c 1 -f -o gpurun_out/k_tc_mxp \
    python tools/perf_run.py mxp 65536 1e-5 > gpurun_out/k_tc_mxp.out 2>&1; echo native rc=$?
ls -la gpurun_out/*.ncu-rep
