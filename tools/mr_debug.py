import sys, os, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import paper_2410_09819_b200 as m
import workloads as w
from test_gpu_multirank import _ranks, _run
n, nb = 1024, 256
P = int(os.environ.get("P", "2"))
A = w.plgsy(n, seed=17)
Lref = np.linalg.cholesky(A)
for trial in range(2):
    plans = _ranks(n, nb, P)
    for pl in plans:
        pl.set("profile", 1)
        if os.environ.get("DS"): pl.set("debug_sync", int(os.environ["DS"]))
    As = [torch.tensor(np.ascontiguousarray(A.T), device="cuda").T for _ in range(P)]
    res = _run(plans, lambda r, pl: pl.factor_device(As[r], stream_from_torch=False))
    torch.cuda.synchronize()
    print("trial", trial, "infos", res)
    for r, pl in enumerate(plans):
        d = pl.sched_diagnostics()
        print(r, {k: v for k, v in d.items() if k != "potrf_timeline_ms"}, d.get("potrf_timeline_ms"))
    Lr = [np.tril(a.cpu().numpy()) for a in As]
    for r in range(P):
        for j in range(n // nb):
            for i in range(j, n // nb):
                blk = Lr[r][i*nb:(i+1)*nb, j*nb:(j+1)*nb]; ref = Lref[i*nb:(i+1)*nb, j*nb:(j+1)*nb]
                raw = np.tril(A)[i*nb:(i+1)*nb, j*nb:(j+1)*nb]
                print(r, (i, j), "own", i % P == r, "err %.2e |blk| %.2e |ref| %.2e raw? %s" % (
                    np.max(np.abs(blk - ref)), np.max(np.abs(blk)), np.max(np.abs(ref)), np.array_equal(blk, raw)))
