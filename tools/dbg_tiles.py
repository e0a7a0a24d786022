import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import oracle, workloads as w
import paper_2410_09819_b200 as m
from gpu_util import gpu_factor
from test_gpu_tiles import pack, unpack, NAT
n, nb = int(sys.argv[1]), int(sys.argv[2])
xy = w.matern_locations(n, seed=1); S = w.matern_cov(xy, 1.0, 0.02627)
pmap = oracle.plan(S, nb, 1e-5)
Ld, info, ld, _ = gpu_factor(S, nb, pmap, attrs=NAT)
tiles, scales = pack(S, nb, pmap)
sc_in = scales.copy()
plan = m.Plan(n, nb, pmap)
for k, v in NAT.items(): plan.set(k, v)
print("info", plan.factor_tiles(tiles, scales), "logdet", plan.logdet(), ld)
Lt = unpack(tiles, scales, n, nb, pmap)
Nt = n // nb
for j in range(Nt):
    for i in range(j, Nt):
        t = oracle.tile_index(Nt, i, j)
        d = np.max(np.abs(Lt[i*nb:(i+1)*nb, j*nb:(j+1)*nb] - Ld[i*nb:(i+1)*nb, j*nb:(j+1)*nb]))
        mx = np.max(np.abs(Ld[i*nb:(i+1)*nb, j*nb:(j+1)*nb]))
        if d > 0: print((i, j), "p", pmap[t], "diff", d, "max", mx, "scale in/out", sc_in[t], scales[t])
