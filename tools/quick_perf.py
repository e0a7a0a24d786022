"""Quick timing of the device path vs cuSOLVER (torch.linalg.cholesky) -- dev tool."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2410_09819_b200 as m

for spec in sys.argv[1:]:
    n, nb = map(int, spec.split(":"))
    A = torch.empty((n, n), dtype=torch.float64, device="cuda").T
    pmap = None
    if os.environ.get("MXP"):
        import workloads as w
        xy = w.matern_locations(n, seed=1)
        m.generate_matern_device(A, xy, 1.0, float(os.environ.get("RANGE", "0.02627")))
        pmap, _ = m.precision_map_from_matrix_device(A, nb, float(os.environ["MXP"]))
        import numpy as np
        Ntt = n // nb
        off = [pmap[i] for i in range(len(pmap))]
        print("   map fractions (FP64,FP32,FP16,FP8):", [round(float(np.mean(pmap == c)), 3) for c in range(4)], flush=True)
    else:
        m.generate_plgsy_device(A, 42)
    plan = m.Plan(n, nb, pmap)
    if os.environ.get("TC") is not None:
        plan.set("tc_engine", int(os.environ["TC"]))
    if os.environ.get("KC"):
        plan.set("splitk_tiles", int(os.environ["KC"]))
    if os.environ.get("PROBE"):
        plan.set("debug_sync", 2)
    plan.use_torch_workspace()
    plan.set("profile", 1)
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
    for k, (nl, ms, fl) in plan.kernel_stats().items():
        print(f"    {k:6s} launches={nl:5d} ms={ms:9.2f} TF/s={(fl/(ms/1e3)/1e12 if ms and fl else 0):6.2f}", flush=True)
    d = plan.sched_diagnostics()
    if d:
        pot = d.pop("potrf_timeline_ms")
        print("    sched", {k: (round(v, 2) if isinstance(v, float) else v) for k, v in d.items()}, flush=True)
        durs = [e - w for (s0, w, e) in pot]
        gaps = [pot[i][1] - pot[i - 1][2] for i in range(1, len(pot))]
        print(f"    KC={plan.get('splitk_tiles')} busy/CTA gemm {d['gemm_busy_ms']/d['ctas']:.1f} ms wait {d['gemm_wait_ms']/d['ctas']:.1f} trsm {d['trsm_busy_ms']/d['ctas']:.1f} ms", flush=True)
        print(f"    potrf: mean dur {sum(durs)/len(durs):.3f} ms, max {max(durs):.3f}; last 6 (start,ready,end): "
              + str([tuple(round(x, 2) for x in t) for t in pot[-6:]]), flush=True)
        print(f"    potrf ready-wait gaps (ms) first 8: {[round(g,3) for g in gaps[:8]]} last 8: {[round(g,3) for g in gaps[-8:]]}", flush=True)
    del B, L
    if os.environ.get("NO_CUSOLVER"):
        continue
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
