#!/bin/bash
# ncu of the MxP static-schedule kernel in the GEMM-only probe (second launch = warm)
PROBE=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sched -s 1 -c 1 -o gpurun_out/ncu_mxp_probe python tools/ncu_mxp.py 16384 1024 1e-8 > gpurun_out/ncu_mxp.log 2>&1
echo rc=$?
tail -3 gpurun_out/ncu_mxp.log
# same probe timed without the profiler (CUDA events in the library)
PROBE=1 timeout 300 python - <<'PY'
import sys, os, time
sys.path.insert(0, "."); sys.argv = ["x", "16384", "1024", "1e-8"]
import numpy as np, torch, paper_2410_09819_b200 as m, workloads as w
n, nb = 16384, 1024
xy = w.matern_locations(n, seed=1); xyd = torch.as_tensor(xy, device="cuda").contiguous()
for eps in (1e-8, 1e-5, 0):
    pmap = m.precision_map_matern_device(xyd, nb, eps, 1.0, 0.02627)[0] if eps else None
    pl = m.Plan(n, nb, pmap); pl.set("debug_sync", 2); pl.set("profile", 1)
    for i in range(3):
        pl.factor_matern(xyd, 1.0, 0.02627); torch.cuda.synchronize()
    ks = pl.kernel_stats()["chain"]
    print("probe eps", eps, "chain ms", ks[1], "TF/s (all GEMM flops incl. garbage)", ks[2] / (ks[1] / 1e3) / 1e12)
PY
