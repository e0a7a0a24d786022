python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/clk.csv &
SMI=$!
for kc in 1 2 4 8; do KC=$kc NO_CUSOLVER=1 timeout 300 python tools/quick_perf.py 65536:1024 2>&1 | grep -E "TF/s probe|KC=|potrf: mean"; done
kill $SMI
sort gpurun_out/clk.csv | uniq -c | sort -rn | head -8
