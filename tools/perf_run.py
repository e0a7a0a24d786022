"""One factorization for profiling (ncu) or quick timing.

    python tools/perf_run.py c2 [n] [nb]            plgsy FP64, Ozaki engine, device-resident
    python tools/perf_run.py mxp [n] [eps] [nb]     Matern weak, map from eps, generated tiles
Prints the wall time of the last of `reps` runs (CUDA events).  Test/dev tool only.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2410_09819_b200 as m  # noqa: E402
import workloads as w  # noqa: E402


def report(plan):
    if os.environ.get("PROFILE") != "1":
        return
    d = plan.sched_diagnostics()
    tl = d.pop("potrf_timeline_ms", None)
    if tl:  # per column: POTRF compute (end - inputs ready) and the gap to the next column's inputs
        comp = [e - w for (_, w, e) in tl]
        gap = [tl[k + 1][1] - tl[k][2] for k in range(len(tl) - 1)]
        q = lambda v: [round(sorted(v)[int(f * (len(v) - 1))], 2) for f in (0.1, 0.5, 0.9)]
        print("potrf compute ms p10/50/90:", q(comp), "sum", round(sum(comp), 1),
              "| inputs-ready gap after previous POTRF p10/50/90:", q(gap), "sum", round(sum(gap), 1),
              "| last 8 columns (compute, gap):", [(round(comp[k], 2), round(gap[k], 2)) for k in range(len(gap) - 8, len(gap))])
    ctas = max(1, d.get("ctas", 1))
    print("sched:", {k: (round(v, 1) if isinstance(v, float) else v) for k, v in d.items()})
    print("per-CTA ms: gemm busy %.1f wait %.1f, trsm busy %.1f wait %.1f" % (
        d["gemm_busy_ms"] / ctas, d["gemm_wait_ms"] / ctas, d["trsm_busy_ms"] / ctas, d["trsm_wait_ms"] / ctas))
    print("ozaki loop ms per CTA:", {k: round(v / ctas, 1) for k, v in d["ozaki_ms"].items()})
    print("native ms per CTA:", {k: round(v / ctas, 1) for k, v in d["native_ms"].items()})
    print("gemm busy ms per CTA by precision:", {k: round(v / ctas, 1) for k, v in d["gemm_busy_ms_by_precision"].items()},
          "tasks:", d["gemm_tasks_by_precision"])
    print("kernels:", plan.kernel_stats())


def main():
    mode = sys.argv[1]
    reps = int(os.environ.get("REPS", "1"))
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if mode == "c2":
        n = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
        nb = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
        A0 = torch.empty((n, n), dtype=torch.float64, device="cuda").T
        m.generate_plgsy_device(A0, seed=42)
        A = torch.empty_like(A0)
        plan = m.Plan(n, nb)
        if "SPLITK" in os.environ:
            plan.set("splitk_tiles", int(os.environ["SPLITK"]))
        plan.set("profile", int(os.environ.get("PROFILE", "0")))
        plan.set("fp64_engine", int(os.environ.get("ENGINE", "1")))
        if "OZ_PF" in os.environ:
            plan.set("oz_prefetch", int(os.environ["OZ_PF"]))
        for r in range(reps):
            A.copy_(A0)
            ev0.record()
            info = plan.factor_device(A)
            ev1.record()
            torch.cuda.synchronize()
        print(f"c2 n={n} nb={nb} info={info} ms={ev0.elapsed_time(ev1):.1f} "
              f"TF/s={n ** 3 / 3 / ev0.elapsed_time(ev1) / 1e9:.2f} engine={plan.get('fp64_engine_used')}")
        report(plan)
        if os.environ.get("SOLVE") == "1":  # forward solve / log-likelihood on the resident factor
            y = torch.randn(n, dtype=torch.float64, device="cuda")
            for r in range(3):
                ev0.record()
                ll = plan.loglik(y)
                ev1.record()
                torch.cuda.synchronize()
            print(f"loglik ms={ev0.elapsed_time(ev1):.2f} GB/s={(n * n / 2 * 8) / ev0.elapsed_time(ev1) / 1e6:.0f} ll={ll:.6e}")
    else:
        n = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
        eps = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-5
        nb = int(sys.argv[4]) if len(sys.argv) > 4 else 1024
        a = float(os.environ.get("RANGE", "0.02627"))
        xy = torch.tensor(w.matern_locations(n, seed=1), device="cuda")
        pmap, _ = m.precision_map_matern_device(xy, nb, eps, 1.0, a)
        plan = m.Plan(n, nb, pmap)
        if "OZ_PF" in os.environ:
            plan.set("oz_prefetch", int(os.environ["OZ_PF"]))
        if "SPLITK" in os.environ:
            plan.set("splitk_tiles", int(os.environ["SPLITK"]))
        plan.set("profile", int(os.environ.get("PROFILE", "0")))
        plan.set("fp64_engine", 1)
        for r in range(reps):
            ev0.record()
            info = plan.factor_matern(xy, 1.0, a)
            ev1.record()
            torch.cuda.synchronize()
        print(f"mxp n={n} eps={eps} info={info} ms={ev0.elapsed_time(ev1):.1f} "
              f"TF/s={n ** 3 / 3 / ev0.elapsed_time(ev1) / 1e9:.2f} tc_engine={plan.get('tc_engine_used')}")
        report(plan)


if __name__ == "__main__":
    main()
