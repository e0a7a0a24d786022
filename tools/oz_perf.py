"""Dev tool: FP64 engine comparison (DMMA vs Ozaki int8) on plgsy n x n, device path."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2410_09819_b200 as m

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
engines = [int(x) for x in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["1", "0"])]
slices = int(os.environ.get("S", "8"))
A = torch.empty((n, n), dtype=torch.float64, device="cuda").T
m.generate_plgsy_device(A, 42)
B = torch.empty_like(A.T).T
x = torch.randn(n, 1, dtype=torch.float64, device="cuda")
Ax = A @ x
nA = torch.linalg.matrix_norm(A, 'fro')
for eng in engines:
    plan = m.Plan(n, nb)
    plan.set("fp64_engine", eng)
    plan.set("oz_slices", slices)
    if os.environ.get("KC"):
        plan.set("splitk_tiles", int(os.environ["KC"]))
    plan.use_torch_workspace()
    plan.set("profile", 1)
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
    L = torch.tril(B)
    r = (Ax - L @ (L.T @ x)).norm() / (nA * x.norm())
    print(f"engine={eng} used={plan.get('fp64_engine_used')} s={slices} n={n} nb={nb} info={info} "
          f"t={t:.3f}s {n**3/3/t/1e12:.2f} TF/s probe={r.item():.2e} logdet={plan.logdet():.10f}", flush=True)
    for k, (nl, ms, fl) in plan.kernel_stats().items():
        print(f"    {k:6s} launches={nl:5d} ms={ms:9.2f} TF/s={(fl/(ms/1e3)/1e12 if ms and fl else 0):6.2f}", flush=True)
    d = plan.sched_diagnostics()
    if d:
        d.pop("potrf_timeline_ms", None)
        print("    sched", {k: (round(v, 2) if isinstance(v, float) else v) for k, v in d.items()}, flush=True)
    del L
    plan.close()
    torch.cuda.empty_cache()
