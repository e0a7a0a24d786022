#!/bin/bash
# OOC leg only (C2 timed briefly first: the OOC line reports its ratio to it)
mkdir -p gpurun_out
timeout 900 python bench.py --steps 2 --warmup 1 --no-e2e --no-cusolver --no-cpu --no-mxp --no-engine-compare --no-kl \
    > gpurun_out/bench_ooc.json 2> gpurun_out/bench_ooc.err; tail -3 gpurun_out/bench_ooc.err
python - <<'P'
import json
d = json.loads(open("gpurun_out/bench_ooc.json").read().strip().splitlines()[-1])
o = d["ooc"]; t = o.pop("timeline") or {}
for k in ("h2d_done_ms", "d2h_done_ms", "work_done_ms"): t.pop(k, None)
print("C2", d["value"]); print(json.dumps(o)); print(json.dumps(t))
P
