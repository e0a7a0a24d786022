"""Debug helper (GPU box): run one MxP factorization per engine setting and report."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import workloads as w
import paper_2410_09819_b200 as m

def run(n, nb, eps, fp64, tc, gen=False, dbg=0):
    xy = w.matern_locations(n, seed=1)
    xyd = torch.as_tensor(xy, device="cuda").contiguous()
    pmap, _ = m.precision_map_matern_device(xyd, nb, eps, 1.0, 0.02627)
    pl = m.Plan(n, nb, pmap)
    pl.set("fp64_engine", fp64); pl.set("tc_engine", tc)
    if dbg: pl.set("debug_sync", dbg)
    t0 = time.time()
    try:
        if gen:
            info = pl.factor_matern(xyd, 1.0, 0.02627)
        else:
            A = torch.empty((n, n), dtype=torch.float64, device="cuda").T
            m.generate_matern_device(A, xyd, 1.0, 0.02627)
            info = pl.factor_device(A)
        torch.cuda.synchronize()
        print(f"n={n} nb={nb} eps={eps} fp64={fp64} tc={tc} gen={gen} used={pl.get('tc_engine_used')} "
              f"info={info} logdet={pl.logdet():.10f} t={time.time()-t0:.2f}s", flush=True)
    except Exception as e:
        print(f"n={n} nb={nb} eps={eps} fp64={fp64} tc={tc} gen={gen} FAILED: {e}", flush=True)
    pl.close()

if __name__ == "__main__":
    for spec in sys.argv[1:]:
        a = spec.split(",")
        run(int(a[0]), int(a[1]), float(a[2]), int(a[3]), int(a[4]), len(a) > 5 and a[5] == "g",
            int(a[6]) if len(a) > 6 else 0)
