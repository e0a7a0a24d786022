"""Dev tool: C3-like MxP timing (Matern weak, generated in the schedule) per FP64 engine."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import numpy as np
import paper_2410_09819_b200 as m
import workloads as w
n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
nb = 1024
xy = torch.as_tensor(w.matern_locations(n, seed=1), device="cuda").contiguous()
for eps in [None, 1e-8, 1e-5]:
    pmap = None if eps is None else m.precision_map_matern_device(xy, nb, eps, 1.0, 0.02627)[0]
    for eng in (1, 0):
        pl = m.Plan(n, nb, pmap)
        pl.set("fp64_engine", eng)
        pl.use_torch_workspace()
        ts = []
        for r in range(3):
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); info = pl.factor_matern(xy, 1.0, 0.02627); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 1e3)
        t = min(ts[1:])
        print(f"eps={eps} engine={eng} used={pl.get('fp64_engine_used')} n={n} {n**3/3/t/1e12:.1f} TF/s logdet={pl.logdet():.6f}", flush=True)
        pl.close(); torch.cuda.empty_cache()
