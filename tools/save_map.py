import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2410_09819_b200 as m
import workloads as w
n, nb = int(sys.argv[1]), int(sys.argv[2])
xy = w.matern_locations(n, seed=1)
xyd = torch.as_tensor(xy, device="cuda").contiguous()
for eps in (1e-8, 1e-5):
    pmap, f = m.precision_map_matern_device(xyd, nb, eps, 1.0, 0.02627)
    np.save(f"gpurun_out/map_{n}_{nb}_{eps:g}.npy", pmap)
    print(eps, np.bincount(pmap, minlength=4) / len(pmap))
