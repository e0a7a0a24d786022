"""Dev tool: C3-like MxP timing (Matern weak, generated in the schedule) per engine.
usage: python tools/mxp_perf.py n eps1,eps2 tc1,tc3 [fp64_engine]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import numpy as np
import paper_2410_09819_b200 as m
import workloads as w
n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
epss = [float(e) for e in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["1e-8", "1e-5"])]
tcs = [int(t) for t in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["3", "1"])]
eng = int(sys.argv[4]) if len(sys.argv) > 4 else 1
dbg = int(os.environ.get("DBG", "0"))
nb = 1024
xy = torch.as_tensor(w.matern_locations(n, seed=1), device="cuda").contiguous()
for eps in epss:
    pmap = m.precision_map_matern_device(xy, nb, eps, 1.0, 0.02627)[0]
    fr = [round(float(np.mean(pmap == c)), 3) for c in range(4)]
    for tc in tcs:
        pl = m.Plan(n, nb, pmap)
        pl.set("fp64_engine", eng)
        pl.set("tc_engine", tc)
        pl.set("profile", 1)
        if dbg:
            pl.set("debug_sync", dbg)
        ts = []
        for r in range(3):
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); info = pl.factor_matern(xy, 1.0, 0.02627); e1.record(); torch.cuda.synchronize()
            assert dbg == 2 or info == 0, info
            ts.append(e0.elapsed_time(e1) / 1e3)
        t = min(ts[1:])
        print(f"eps={eps} tiles={fr} tc={tc} used={pl.get('tc_engine_used')} fp64={pl.get('fp64_engine_used')} n={n} "
              f"{n**3/3/t/1e12:.1f} TF/s ws={pl.workspace_size()/1e9:.1f} GB img={pl.get('image_bytes')/1e9:.1f} GB "
              f"logdet={(pl.logdet() if dbg != 2 else 0):.9f}", flush=True)
        for kk, (nl, ms, fl) in pl.kernel_stats().items():
            print(f"    {kk:6s} launches={nl:5d} ms={ms:9.2f} TF/s={(fl/(ms/1e3)/1e12 if ms and fl else 0):6.2f}", flush=True)
        d = pl.sched_diagnostics()
        if d:
            d.pop("potrf_timeline_ms", None)
            print("    sched", {k: (round(v, 2) if isinstance(v, float) else v) for k, v in d.items()}, flush=True)
        pl.close(); torch.cuda.empty_cache()
