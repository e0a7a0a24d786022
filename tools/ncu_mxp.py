"""Profiling driver: one warm-up + one profiled factor_matern (MxP map) at n."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2410_09819_b200 as m
import workloads as w
n, nb, eps = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
xy = w.matern_locations(n, seed=1)
xyd = torch.as_tensor(xy, device="cuda").contiguous()
pmap = None
if eps > 0:
    pmap, _ = m.precision_map_matern_device(xyd, nb, eps, 1.0, 0.02627)
    print("fractions", np.bincount(pmap, minlength=4) / len(pmap))
pl = m.Plan(n, nb, pmap)
if os.environ.get("PROBE"):
    pl.set("debug_sync", 2)  # GEMM-throughput probe: every tile Ready, no POTRF/TRSM (values garbage)
for i in range(2):
    info = pl.factor_matern(xyd, 1.0, 0.02627)
    torch.cuda.synchronize()
    if os.environ.get("PROBE"):
        continue
    print("info", info, "logdet", pl.logdet(), "image_bytes", pl.get("image_bytes"))
