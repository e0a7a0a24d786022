"""Quick timing of the device path vs cuSOLVER (torch.linalg.cholesky) -- dev tool."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2410_09819_b200 as m

for spec in sys.argv[1:]:
    n, nb = map(int, spec.split(":"))
    A = torch.empty((n, n), dtype=torch.float64, device="cuda").T
    m.generate_plgsy_device(A, 42)
    plan = m.Plan(n, nb)
    plan.use_torch_workspace()
    B = torch.empty_like(A.T).T
    ts = []
    for r in range(3):
        B.copy_(A)
        torch.cuda.synchronize()
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record()
        info = plan.factor_device(B)
        e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) / 1e3)
    t = min(ts)
    # residual probe
    L = torch.tril(B)
    x = torch.randn(n, 1, dtype=torch.float64, device="cuda")
    r = (A @ x - L @ (L.T @ x)).norm() / (torch.linalg.matrix_norm(A, 2 if n <= 4096 else 'fro') * x.norm())
    print(f"n={n} nb={nb} info={info} t={t:.3f}s {n**3/3/t/1e12:.2f} TF/s probe={r.item():.2e} launches={plan.get('gpu_launches')}", flush=True)
    del B, L
    S = A.T.contiguous()
    ts = []
    for r in range(2):
        torch.cuda.synchronize(); t0 = time.time()
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); Lc, inf = torch.linalg.cholesky_ex(S); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) / 1e3)
        del Lc
    print(f"   cusolver t={min(ts):.3f}s {n**3/3/min(ts)/1e12:.2f} TF/s", flush=True)
    del S, A, plan
    torch.cuda.empty_cache()
