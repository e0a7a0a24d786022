#!/bin/bash
# dev loop on the GPU box: build, a pytest selection ($1), then a short C2 bench line
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/build.log 2>&1; tail -3 gpurun_out/build.log
timeout 1200 python -m pytest -q -m gpu -p no:randomly -x $1 > gpurun_out/pytest_dev.log 2>&1; tail -15 gpurun_out/pytest_dev.log
timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cusolver --no-cpu --no-mxp --no-ooc --no-engine-compare --no-kl \
    > gpurun_out/bench_dev.json 2> gpurun_out/bench_dev.err; tail -c 400 gpurun_out/bench_dev.err
python - <<'P'
import json
d = json.loads(open("gpurun_out/bench_dev.json").read().strip().splitlines()[-1])
print("C2", d["value"], d["unit"], "ms", d["ms_per_step"], "roof", d.get("roofline", {}).get("frac"), "bwd", d.get("check", {}).get("backward_error_fro"), "clk", d.get("clocks"))
P
