import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import paper_2410_09819_b200 as m
import workloads as w
n, nb = 1024, 256
A = w.plgsy(n, seed=17)
Lref = np.linalg.cholesky(A)
def run(name, setup, sft=True):
    pl = m.Plan(n, nb)
    setup(pl)
    Ad = torch.tensor(np.ascontiguousarray(A.T), device="cuda").T
    info = pl.factor_device(Ad, stream_from_torch=sft)
    torch.cuda.synchronize()
    L = np.tril(Ad.cpu().numpy())
    print(name, "info", info, "err %.2e" % np.max(np.abs(L - Lref)), flush=True)
run("plain", lambda p: None)
run("profile", lambda p: p.set("profile", 1))
run("nosft", lambda p: None, sft=False)
run("rank0", lambda p: (p.set("rank", 0), p.set("nranks", 1)))
run("smpart", lambda p: (p.set("sm_first", 0), p.set("sm_count", 148)))
run("smpart74", lambda p: (p.set("sm_first", 0), p.set("sm_count", 74)))
run("smpart74b", lambda p: (p.set("sm_first", 74), p.set("sm_count", 74)))
