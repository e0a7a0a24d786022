python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
PROBE=1 KC=8 NO_CUSOLVER=1 python tools/quick_perf.py 65536:1024 2>&1 | grep -E "TF/s probe|KC="
PROBE=1 KC=8 NO_CUSOLVER=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sched -s 1 -c 1 -o gpurun_out/prof_sched -f python tools/quick_perf.py 16384:1024 > gpurun_out/ncu_sched.log 2>&1; tail -2 gpurun_out/ncu_sched.log
