#!/usr/bin/env python
"""Benchmark: factorization TFLOP/s (n^3/3) of the left-looking tile Cholesky
(arxiv 2410.09819) on B200, vs cuSOLVER potrf and the roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

FP64 engine (--fp64-engine): "ozaki" (default) runs the FP64 GEMM/SYRK updates
as exact int8 slice products on the tcgen05 tensor cores (Ozaki scheme I, 8
slices = 55-bit operands, int32/fp64 accumulation) -- its
backward error is checked every run and reported beside the native FP64
tensor-pipe (DMMA) engine's, which is also timed (fp64_engines).

Workload (BASELINE.json configs[1], "C2"): n = 65536, nb = 1024, FP64,
PLASMA-plgsy random SPD (seed 42, generated on the device by the same counter
hash as workloads/), in-core on one B200.  A step = one full factorization
(restore the input from a resident copy, then mxp_chol_factor_device); inputs
(34 GB) are far larger than L2 (126 MB).  Timed with CUDA events on the
plan's stream, barrier + synchronize on both sides, max over ranks.

`e2e` is the same metric through the host API mxp_chol_factor on a pinned host
matrix (H2D + factor + D2H inside the timed region, every step).
`--impl reference` times the CPU oracle (oracle/, test infrastructure) on a
bounded sample of the same workload family on the host cores.

For N > 1 the ranks (one process per GPU, torchrun) factor ONE matrix
together: tile row m belongs to rank m mod N, finished tiles are pushed to the
peers' pools by the copy engines over NVLink (IPC-mapped workspaces, handles
exchanged through torch.distributed), value = (n^3/3) / max-over-ranks step
time (strong scaling).  With fewer visible GPUs than ranks the ranks share
GPU 0 with split SMs (functional check only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
# every stream its own hardware queue: streams parked on cuStreamWaitValue32
# (tile pushes, start barrier) must not block others sharing their queue
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, ROOT)

METRIC = "factorization TFLOP/s (n^3/3) at 1/2/4/8 B200 vs cuSOLVER potrf & roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--size", dest="n", type=int, default=65536)  # not "--n": torchrun prefix-matches it
    ap.add_argument("--nb", type=int, default=1024)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cusolver", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-mxp", action="store_true")
    ap.add_argument("--mxp-n", type=int, default=131072)
    ap.add_argument("--mxp-eps", type=float, nargs="*", default=[1e-5, 1e-6, 1e-7, 1e-8, 1e-9])
    ap.add_argument("--kl-n", type=int, default=32768)
    ap.add_argument("--no-kl", action="store_true")
    ap.add_argument("--no-ooc", action="store_true")
    ap.add_argument("--ooc-n", type=int, default=98304)
    ap.add_argument("--ooc-frac", type=float, default=0.65)
    ap.add_argument("--fp64-engine", default="ozaki", choices=["dmma", "ozaki"],
                    help="GEMM/SYRK engine of FP64 tiles: FP64 tensor pipe (DMMA) or Ozaki-I on int8 tcgen05")
    ap.add_argument("--oz-slices", type=int, default=7)
    ap.add_argument("--no-engine-compare", action="store_true")
    return ap.parse_args()


def progress(what):
    """leg markers on stderr (the JSON line stays the only stdout line)"""
    print(f"[bench] {time.strftime('%H:%M:%S')} done: {what}", file=sys.stderr, flush=True)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = []
        with open(self.f.name) as fh:
            for line in fh:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        loaded = [s for s in sm if s > 0.5 * (max(mx) if mx else 1)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


def cpu_oracle_sample(n=2048, nb=256, seed=42):
    """Time the CPU oracle (as it stands) on a bounded sample of the workload."""
    import oracle
    import workloads as w
    A = w.plgsy(n, seed)
    oracle.build()
    t0 = time.perf_counter()
    L, info = oracle.factor(A, nb)
    t = time.perf_counter() - t0
    assert info == 0
    return {"value": n ** 3 / 3 / t / 1e12, "unit": "TFLOP/s", "cores": os.cpu_count(),
            "kind": "oracle", "seconds": t,
            "sample": f"oracle.factor (plain C fp64, OpenMP over a column's tasks) on plgsy "
                      f"n={n} nb={nb} FP64, the same matrix family at a size the oracle finishes in "
                      f"seconds; rate = (n^3/3)/t"}


def cpu_baselines(seed=42):
    """SURVEY 8(d) oracle timing table on the host cores: C1 exactly, FP64 and 4-precision Matern
    at n = 4096, plus LAPACK dpotrf (numpy/OpenBLAS) at n = 16384 as the optimized-CPU point.
    Rates in GFLOP/s = (n^3/3)/t; the larger configs are extrapolated by n^3 in DESIGN.md."""
    import numpy as np

    import oracle
    import workloads as w
    oracle.build()
    out = {"cores": os.cpu_count()}

    def t_oracle(A, nb, pmap=None):
        t0 = time.perf_counter()
        _, info = oracle.factor(A, nb, pmap)
        assert info == 0
        return time.perf_counter() - t0
    A = w.kms(1024, 0.5)
    t = t_oracle(A, 256)
    out["c1_oracle"] = {"n": 1024, "nb": 256, "s": t, "gflops": 1024 ** 3 / 3 / t / 1e9}
    A = w.plgsy(4096, seed)
    t = t_oracle(A, 256)
    out["oracle_fp64_n4096"] = {"nb": 256, "s": t, "gflops": 4096 ** 3 / 3 / t / 1e9}
    xy = w.matern_locations(4096, seed=1)
    S = w.matern_cov(xy, 1.0, 0.02627)
    pm = oracle.plan(S, 256, 1e-5)
    t = t_oracle(S, 256, pm)
    out["oracle_mxp_n4096"] = {"nb": 256, "eps": 1e-5, "s": t, "gflops": 4096 ** 3 / 3 / t / 1e9}
    A = w.plgsy(16384, seed)
    t0 = time.perf_counter()
    np.linalg.cholesky(A)
    t = time.perf_counter() - t0
    try:
        import threadpoolctl
        th = [x.get("num_threads") for x in threadpoolctl.threadpool_info() if x.get("user_api") == "blas"]
    except Exception:
        th = None
    out["lapack_dpotrf_n16384"] = {"s": t, "gflops": 16384 ** 3 / 3 / t / 1e9, "blas_threads": th,
                                   "how": "numpy.linalg.cholesky (LAPACK dpotrf via numpy's BLAS)"}
    return out


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    n, nb = 2048, 256
    times = []
    for i in range(args.warmup + args.steps):
        r = cpu_oracle_sample(n, nb, args.seed)
        if i >= args.warmup:
            times.append(r["seconds"])
    t = sum(times) / len(times)
    value = n ** 3 / 3 / t / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"C2 family (plgsy random SPD, FP64) -- bounded sample n={n} nb={nb} "
                               f"per step on the host cores (the reference arm is the CPU oracle)",
                   "n": n, "nb": nb, "seed": args.seed},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": os.cpu_count(), "kind": "oracle",
                         "sample": f"oracle.factor plgsy n={n} nb={nb} per step"},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def int8_peak():
    """Dense int8 tensor peak: MEASURED_PEAKS.json's sustained bf16 dense figure (k_tc runs for
    seconds inside the step) x the nominal int8:bf16 ratio (2)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return 2.0 * pk["bf16_tflops_sustained"], (
            "2 x MEASURED_PEAKS.json bf16_tflops_sustained (%.1f; the kernel runs for seconds) -- B200 "
            "int8:bf16 dense ratio 2 (4.5 POPS : 2.25 PFLOPS nominal)" % pk["bf16_tflops_sustained"])
    except Exception:
        return 4500.0, "nominal B200 dense int8 4.5 POPS (MEASURED_PEAKS.json absent)"


def load_traffic(nb, engine="dmma"):
    """dram bytes per launch of the dominant kernel from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "ncu_tc_latest.json" if engine == "ozaki" else "ncu_chain_latest.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch"), d
    except Exception:
        return None, None


def residual_fro(A, B, nbk=4096):
    """||A - L L^T||_F / ||A||_F, L = tril(B), by block columns (cuBLAS DGEMM; independent
    of our kernels): the diagonal block once, the blocks below it twice (symmetry)."""
    import torch
    n = A.shape[0]
    ss = 0.0
    for j0 in range(0, n, nbk):
        j1 = min(n, j0 + nbk)
        Lr = torch.tril(B[j0:, :j1], diagonal=j0)           # rows j0.. of L, columns < j1
        R = A[j0:, j0:j1] - Lr @ Lr[: j1 - j0].T             # block column j of A - L L^T, rows >= j0
        ss += R[: j1 - j0].norm().item() ** 2 + 2.0 * R[j1 - j0:].norm().item() ** 2
        del Lr, R
    return ss ** 0.5 / torch.linalg.matrix_norm(A).item()


def mxp_flops_by_precision(pmap, Nt, nb):
    """Per-precision flops of one factorization (SURVEY 8(d) roofline): GEMM (m,k,n) in p(m,k),
    SYRK in FP64, TRSM nb^3 in FP64 (DMMA), POTRF nb^3/3.  Returns {"fp64_gemm", "fp32", "fp16",
    "fp8", "trsm", "potrf"} in flops; they sum to (Nt nb)^3 / 3."""
    import numpy as np
    F = {"fp64_gemm": 0.0, "fp32": 0.0, "fp16": 0.0, "fp8": 0.0, "trsm": 0.0, "potrf": 0.0}
    nb3 = float(nb) ** 3
    key = {0: "fp64_gemm", 1: "fp32", 2: "fp16", 3: "fp8"}
    pm = np.asarray(pmap)
    for k in range(Nt):
        t0 = k * Nt - k * (k - 1) // 2
        F["fp64_gemm"] += k * nb3          # SYRK of the diagonal tile
        F["potrf"] += nb3 / 3
        for m in range(k + 1, Nt):
            F[key[int(pm[t0 + m - k])]] += 2.0 * k * nb3
            F["trsm"] += nb3
    return F


def mxp_roofline(F, peaks):
    """T_compute = sum_p F_p / peak_p; roof = (n^3/3) / T_compute (TFLOP/s)."""
    T = sum(F[k] / (peaks[k] * 1e12) for k in F if F[k] > 0)
    return sum(F.values()) / T / 1e12, T


def ooc_variant_ledgers(m, n, nb, lower, fracs, h2d_measured, d2h_measured, streams=4):
    """N3 (Alg. 3): host-link bytes of the paper's
    OOC variants replayed over the same static task sequence with HBM for `frac` of the lower
    triangle (mxp_ooc_variant_volume; 4 streams), beside the engine's own measured ledger."""
    out = {"how": "mxp_ooc_variant_volume: Alg. 2's tasks dealt to 4 streams, a tile cache of frac x the "
                  "lower triangle; sync/async/V1 have no cache, V2 = LRU cache table (remove_steal), V3 = V2 + "
                  "L_kk pinned until the last TRSM of its column, static = this engine's dead-tile plan, MIN = "
                  "Belady's optimal eviction; bytes are FP64 tiles (replayed ledgers, not executed variants)",
           "engine_measured": {"h2d_bytes": h2d_measured, "d2h_bytes": d2h_measured}}
    for frac in fracs:
        row = {}
        for v in ("sync", "async", "V1", "V2", "V3", "static", "MIN"):
            r = m.ooc_variant_volume(n, nb, v, int(frac * lower), streams)
            row[v] = None if r is None else {"h2d_gb": round(r["h2d_bytes"] / 1e9, 2),
                                             "d2h_gb": round(r["d2h_bytes"] / 1e9, 2),
                                             "total_over_lower": round((r["h2d_bytes"] + r["d2h_bytes"]) / lower, 3)}
        out[f"hbm_{frac:.2f}_of_lower"] = row
    return out


def ooc_timeline_summary(tl, t_total):
    """The paper's Fig. 7 rows (C2G, G2C, Work) as per-column event times of a
    profiled out-of-core run, plus what they say about overlap: a column's loads finishing
    after the previous column's POTRF would stall the schedule on the host link."""
    import numpy as np
    if not tl:
        return None
    h2d, d2h, work = tl["h2d"], tl["d2h"], tl["work"]
    nt = len(work)
    late = [k for k in range(1, nt) if h2d[k] >= 0 and work[k - 1] >= 0 and h2d[k] > work[k - 1]]
    lag = [d2h[k] - work[k] for k in range(nt) if d2h[k] >= 0 and work[k] >= 0]
    return {"columns": nt, "run_ms": t_total * 1e3,
            "h2d_done_ms": [round(x, 3) for x in h2d], "d2h_done_ms": [round(x, 3) for x in d2h],
            "work_done_ms": [round(x, 3) for x in work],
            "columns_loaded_after_previous_potrf": len(late),
            "h2d_all_done_ms": max(h2d), "d2h_lag_after_potrf_ms_median": float(np.median(lag)) if lag else None,
            "how": "CUDA events after each column's H2D loads (C2G), D2H write-backs (G2C) and POTRF (Work), "
                   "ms since the factorization start (mxp_chol_timeline, MXP_ATTR_PROFILE=1)"}


def run_c3(args, m, dev, dev_index, stream, ws, new_plan, allreduce, barrier, dgemm_peak):
    import gc
    import math

    import numpy as np
    import torch

    import workloads as w
    gc.collect()
    torch.cuda.empty_cache()
    nm, nbm, theta = args.mxp_n, args.nb, (1.0, 0.02627, 0.5)
    Nt = -(-nm // nbm)
    xy = w.matern_locations(nm, seed=1)
    xyd = torch.as_tensor(xy, device=dev).contiguous()
    gz = torch.Generator(device=dev).manual_seed(2)
    z = torch.randn(nm, dtype=torch.float64, device=dev, generator=gz)
    flops_m = nm ** 3 / 3
    out = {"workload": f"C3: Matern nu=0.5 theta=(1, 0.02627, 0.5) (weak), n={nm}, nb={nbm}, Morton-sorted "
                       f"uniform locations (seed 1), tiles generated on the device inside the schedule",
           "maps": {}}
    const = -0.5 * nm * math.log(2 * math.pi)

    # ---- independent FP64 reference: cuSOLVER potrf (upper) on the dense matrix (137 GB), in its
    #      own process (a cuSOLVER fault must not poison this context); it also returns y = Sigma z
    y = None
    cus = None
    if ws == 1:
        import subprocess
        import tempfile
        gc.collect()
        torch.cuda.empty_cache()
        tmp = os.path.join(tempfile.mkdtemp(), "c3_ref.npz")
        try:
            r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "cusolver_c3.py"), str(nm), str(theta[1]),
                                tmp], capture_output=True, text=True, timeout=600)
            if r.returncode == 0:
                d = np.load(tmp)
                meta = json.loads(str(d["meta"]))
                y = torch.as_tensor(d["y"], device=dev)
                cus = dict(meta, loglik_y0=const - 0.5 * meta["logdet"],
                           loglik_y=const - 0.5 * meta["logdet"] - 0.5 * meta["quad_form"],
                           how="cusolverDnXpotrf (upper, fp64) on the dense generated covariance in a child "
                               "process; logdet from diag(U); y^T Sigma^-1 y by cusolverDnXpotrs; y = Sigma z, "
                               "z seeded normal (seed 2), computed before the factorization")
            else:
                cus = {"error": (r.stderr or r.stdout)[-300:]}
        except Exception as e:  # noqa -- a library baseline must not abort our measurement
            cus = {"error": repr(e)[:300]}
    out["cusolver_fp64"] = cus
    if y is None:
        y = torch.randn(nm, dtype=torch.float64, device=dev, generator=torch.Generator(device=dev).manual_seed(3))

    def run(pmap, reps, fp64_engine=None):
        pl = new_plan(nm, nbm, pmap, engine=fp64_engine)
        pl.set("profile", 0)
        ts = []
        for i in range(reps):
            torch.cuda.synchronize()
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            inf = pl.factor_matern(xyd, theta[0], theta[1])
            e1.record(stream)
            torch.cuda.synchronize()
            assert inf == 0, inf
            ts.append(allreduce(e0.elapsed_time(e1) / 1e3, "max"))
        r = {"t": min(ts[1:] if len(ts) > 1 else ts), "logdet": pl.logdet(),
             "ws_gb": pl.workspace_size() / 1e9, "img_gb": pl.get("image_bytes") / 1e9,
             "fp64_engine": "ozaki" if pl.get("fp64_engine_used") == 1 else "dmma",
             "tc_engine": pl.get("tc_engine_used"), "compact": pl.get("compact_used"),
             "slots": pl.get("pool_slots")}
        if ws == 1:
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            r["loglik_y"] = pl.loglik(y)
            e1.record(stream)
            torch.cuda.synchronize()
            r["solve_ms"] = e0.elapsed_time(e1)
        pl.close()
        del pl
        gc.collect()
        torch.cuda.empty_cache()
        return r

    reps = 2  # one warm-up + one timed factorization per configuration (bounded bench time)
    r64 = run(None, reps)
    ll64 = const - 0.5 * r64["logdet"]
    out["fp64"] = {"tflops": flops_m / r64["t"] / 1e12, "ms": r64["t"] * 1e3, "logdet": r64["logdet"],
                   "engine": r64["fp64_engine"], "loglik_y0": ll64, "loglik_y": r64.get("loglik_y")}
    if r64.get("solve_ms"):
        lower_bytes = Nt * (Nt + 1) // 2 * nbm * nbm * 8
        out["fp64"]["forward_solve"] = {
            "ms": r64["solve_ms"], "gbs": lower_bytes / (r64["solve_ms"] / 1e3) / 1e9,
            "how": "mxp_chol_loglik(y): forward solve L z = y (every lower tile read once) + ||z||^2"}
    if cus and "logdet" in cus:
        out["fp64"]["loglik_y0_rel_err_vs_cusolver"] = abs(ll64 - cus["loglik_y0"]) / abs(cus["loglik_y0"])
        if r64.get("loglik_y") is not None:
            out["fp64"]["loglik_y_rel_err_vs_cusolver"] = abs(r64["loglik_y"] - cus["loglik_y"]) / abs(cus["loglik_y"])
    best_fp64 = max(out["fp64"]["tflops"], (cus or {}).get("tflops") or 0.0)
    # measured sustained peaks for the per-precision roofline: FP64 GEMM/SYRK on
    # the int8 pipe (s(s+1)/2 products) or DMMA; FP32 = 3 fp16 products (h h + h l + l h); FP16 = bf16
    # dense; FP8 = 2x; TRSM / POTRF on DMMA (live DGEMM)
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            bf16 = json.load(f)["bf16_tflops_sustained"]
    except Exception:
        bf16 = 2250.0 * 0.6
    npairs = args.oz_slices * (args.oz_slices + 1) // 2
    peaks = {"fp64_gemm": 2 * bf16 / npairs, "fp32": bf16 / 3, "fp16": bf16, "fp8": 2 * bf16, "trsm": dgemm_peak,
             "potrf": dgemm_peak}
    g16 = {}
    for eps in args.mxp_eps:
        pmap, _ = m.precision_map_matern_device(xyd, nbm, eps, theta[0], theta[1])
        r = run(pmap, reps)
        llm = const - 0.5 * r["logdet"]
        F = mxp_flops_by_precision(pmap, Nt, nbm)
        pk = dict(peaks)
        if r["fp64_engine"] == "dmma":
            pk["fp64_gemm"] = dgemm_peak
        roof, _ = mxp_roofline(F, pk)
        tfl = flops_m / r["t"] / 1e12
        e = {"tflops": tfl, "ms": r["t"] * 1e3, "speedup_vs_fp64": out["fp64"]["tflops"] and tfl / out["fp64"]["tflops"],
             "speedup_vs_best_fp64": tfl / best_fp64,
             "engines": {"fp64": r["fp64_engine"], "below_fp64": {3: "native (kind::f16/f8f6f4)", 1: "tf32 images",
                                                                  2: "tf32 registers", 0: "dmma"}.get(r["tc_engine"])},
             "compact_pool": bool(r["compact"]), "fp64_pool_slots": r["slots"], "tiles": Nt * (Nt + 1) // 2,
             "workspace_gb": round(r["ws_gb"], 2),
             "image_gb": round(r["img_gb"], 2),
             "tile_fractions_fp64_fp32_fp16_fp8": [round(float(np.mean(pmap == c)), 4) for c in range(4)],
             "flop_fractions": {k: round(v / flops_m, 4) for k, v in F.items()},
             "roofline": {"roof_tflops": roof, "frac": tfl / roof,
                          "how": "roof = (n^3/3) / sum_p F_p/peak_p; peaks: FP64 GEMM = 2 x bf16 sustained / "
                                 f"{npairs} (Ozaki, s={args.oz_slices}) or live DGEMM, FP32 = bf16/3, FP16 = bf16, FP8 = 2 x bf16, TRSM/POTRF = DGEMM"},
             "loglik_y0_rel_err": abs(llm - ll64) / abs(ll64), "logdet_abs_diff": abs(r["logdet"] - r64["logdet"]),
             "kl_eq3": ll64 - llm}
        if r.get("loglik_y") is not None and r64.get("loglik_y") is not None:
            e["loglik_y_rel_err"] = abs(r["loglik_y"] - r64["loglik_y"]) / abs(r64["loglik_y"])
        if cus and "logdet" in cus:
            e["loglik_y0_rel_err_vs_cusolver"] = abs(llm - cus["loglik_y0"]) / abs(cus["loglik_y0"])
            if r.get("loglik_y") is not None:
                e["loglik_y_rel_err_vs_cusolver"] = abs(r["loglik_y"] - cus["loglik_y"]) / abs(cus["loglik_y"])
        ok = e["loglik_y0_rel_err"] <= 1e-6 and e.get("loglik_y_rel_err", 0.0) <= 1e-6
        e["meets_g16"] = ok
        if ok:
            g16[eps] = e
        out["maps"][f"{eps:g}"] = e
    if g16:
        eps_best = max(g16)
        out["largest_eps_meeting_g16"] = {"eps": eps_best, "tflops": g16[eps_best]["tflops"],
                                          "speedup_vs_best_fp64": g16[eps_best]["speedup_vs_best_fp64"],
                                          "g16": "|l_MxP - l_FP64| / |l_FP64| <= 1e-6 at y = 0 and y = Sigma z"}
    out["note"] = ("TFLOP/s = (n^3/3)/t, t = one factorization incl. fused generation (1 warm-up + 1 timed); "
                   "loglik vs our FP64 run of the same pipeline and vs cuSOLVER")
    return out


def run_kl_sweep(args, m, dev, new_plan):
    """N1: Eq. 3 KL = l_FP64(theta;0) - l_MxP(theta;0) and l at y = Sigma z over the
    three correlations x eps at n = args.kl_n (the C3 size is the eps sweep of run_c3)."""
    import gc
    import math

    import torch

    import workloads as w
    n, nb = args.kl_n, args.nb
    xy = w.matern_locations(n, seed=1)
    xyd = torch.as_tensor(xy, device=dev).contiguous()
    z = torch.randn(n, dtype=torch.float64, device=dev, generator=torch.Generator(device=dev).manual_seed(2))
    const = -0.5 * n * math.log(2 * math.pi)
    rows = []
    for name, a in (("weak", 0.02627), ("medium", 0.078809), ("strong", 0.210158)):
        A = torch.empty((n, n), dtype=torch.float64, device=dev).T
        m.generate_matern_device(A, xyd, 1.0, a)
        y = A @ z
        del A
        torch.cuda.empty_cache()
        res = {}
        for eps in [None] + list(args.mxp_eps):
            pmap = None if eps is None else m.precision_map_matern_device(xyd, nb, eps, 1.0, a)[0]
            pl = new_plan(n, nb, pmap)
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t0.record()
            info = pl.factor_matern(xyd, 1.0, a)
            t1.record()
            torch.cuda.synchronize()
            res[eps] = (info, pl.logdet() if info == 0 else None, pl.loglik(y) if info == 0 else None,
                        t0.elapsed_time(t1))
            pl.close()
            gc.collect()
            torch.cuda.empty_cache()
        i64, ld64, lly64, _ = res[None]
        l0 = const - 0.5 * ld64
        for eps in args.mxp_eps:
            info, ld, lly, ms = res[eps]
            if info != 0:
                rows.append({"theta": name, "range_a": a, "eps": eps, "info": info})
                continue
            la = const - 0.5 * ld
            kl = l0 - la
            rows.append({"theta": name, "range_a": a, "eps": eps, "kl_eq3": kl,
                         "log10_abs_kl": math.log10(abs(kl)) if kl else None,
                         "loglik_y0_rel_err": abs(la - l0) / abs(l0),
                         "loglik_y_rel_err": abs(lly - lly64) / abs(lly64), "ms": ms})
    return {"n": n, "nb": nb, "rows": rows,
            "how": "Eq. 3 KL = l0(theta;0) - la(theta;0) (G17, signed), l0 = FP64 factorization, la = MxP map "
                   "at eps; l(y) at y = Sigma z; tiles generated in the schedule"}


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2410_09819_b200 as m

    ws, rank, local = dist_env()
    # one process per GPU; with fewer visible GPUs than ranks (a test setup)
    # the ranks share GPU 0 and split its SMs
    coloc = ws > 1 and torch.cuda.device_count() < ws
    dev_index = 0 if coloc else local
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    if ws > 1:
        if coloc:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    red_dev = "cpu" if coloc else dev

    def barrier():
        if ws > 1:
            dist.barrier()

    def allreduce(x, op="max"):
        if ws == 1:
            return x
        t = torch.tensor([float(x)], device=red_dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
        return t.item()

    ENG = {"dmma": 0, "ozaki": 1}

    def new_plan(nn, nbb, pmap=None, engine=None):
        pl = m.Plan(nn, nbb, pmap)
        pl.set("device", dev_index)
        pl.set("fp64_engine", ENG[engine or args.fp64_engine])
        pl.set("oz_slices", args.oz_slices)
        if ws > 1:
            pl.connect(rank, ws, sm_partition=coloc)  # row-cyclic ranks, IPC-mapped peer pools
        else:
            pl.use_torch_workspace(dev)
        return pl

    n, nb = args.n, args.nb
    flops = n ** 3 / 3

    m.lib()  # the in-tree CUDA library must load: no fallback path exists
    stream = torch.cuda.current_stream()
    A = torch.empty((n, n), dtype=torch.float64, device=dev).T  # column-major
    m.generate_plgsy_device(A, seed=args.seed, stream=stream.cuda_stream)
    B = torch.empty((n, n), dtype=torch.float64, device=dev).T
    plan = new_plan(n, nb)
    plan.set("profile", 1)

    def step():
        B.copy_(A)
        return plan.factor_device(B)

    for _ in range(args.warmup):
        info = step()
        assert info == 0, info
    clocks = Clocks(dev_index)
    clocks.start()
    stats_acc = {}
    launches = 0
    barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        info = step()
        assert info == 0, info
        launches += plan.get("gpu_launches") + 0
        for k, (nl, ms, fl) in plan.kernel_stats().items():
            a = stats_acc.setdefault(k, [0, 0.0, 0.0])
            a[0] += nl
            a[1] += ms
            a[2] += fl
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ck = clocks.stop()
    t_step = allreduce(ev0.elapsed_time(ev1) / 1e3 / args.steps, "max")
    launches = int(allreduce(launches, "sum"))
    value = flops / t_step / 1e12  # one n x n factorization per step, over all ranks

    progress("C2 timed")
    # accuracy of the last factor: the full backward error ||A - L L^T||_F / ||A||_F (blockwise
    # cuBLAS DGEMM, independent of our kernels) and the randomized probe ||(A - L L^T) x|| / ||A x||
    backward_error = residual_fro(A, B) if ws == 1 else None
    L = torch.tril(B)
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    x = torch.randn(n, 4, dtype=torch.float64, device=dev, generator=g)
    Ax = A @ x
    probe = ((Ax - L @ (L.T @ x)).norm() / Ax.norm()).item()
    del L, x, Ax
    logdet = plan.logdet()
    sched = plan.sched_diagnostics()
    if sched:
        pot = sched.pop("potrf_timeline_ms")
        sched["potrf_mean_ms"] = sum(e - w for (_, w, e) in pot) / len(pot)
        for key in ("gemm_busy_ms", "gemm_wait_ms", "trsm_busy_ms", "trsm_wait_ms"):
            sched[key + "_per_cta"] = sched.pop(key) / max(sched["ctas"], 1)

    engine_used = "ozaki" if plan.get("fp64_engine_used") == 1 else "dmma"

    progress("probe")
    # the other FP64 engine on the same input (same step, fewer reps)
    engines = {engine_used: {"tflops": value, "ms": t_step * 1e3, "backward_error_fro": backward_error,
                             "backward_error_probe": probe, "logdet": logdet}}
    if not args.no_engine_compare:
        other = "dmma" if engine_used == "ozaki" else "ozaki"
        pl2 = new_plan(n, nb, engine=other)
        ts = []
        for i in range(3):
            B.copy_(A)
            torch.cuda.synchronize()
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            inf = pl2.factor_device(B)
            e1.record(stream)
            torch.cuda.synchronize()
            assert inf == 0, inf
            if i:
                ts.append(allreduce(e0.elapsed_time(e1) / 1e3, "max"))
        be2 = residual_fro(A, B) if ws == 1 else None
        L2 = torch.tril(B)
        x2 = torch.randn(n, 4, dtype=torch.float64, device=dev, generator=torch.Generator(device=dev).manual_seed(7))
        Ax2 = A @ x2
        pr2 = ((Ax2 - L2 @ (L2.T @ x2)).norm() / Ax2.norm()).item()
        del L2, x2, Ax2
        used2 = "ozaki" if pl2.get("fp64_engine_used") == 1 else "dmma"
        engines[used2] = {"tflops": flops / min(ts) / 1e12, "ms": min(ts) * 1e3, "backward_error_fro": be2,
                          "backward_error_probe": pr2, "logdet": pl2.logdet()}
        pl2.close()
        del pl2
        torch.cuda.empty_cache()
    if "ozaki" in engines:
        engines["ozaki"]["slices"] = args.oz_slices
        engines["ozaki"]["what"] = ("Ozaki scheme I: FP64 tiles split exactly into int8 slices (row scales), "
                                    "s(s+1)/2 int8 tcgen05 GEMMs per tile product, exact int32 TMEM "
                                    "accumulation, fp64 combination per tile of K")

    progress("engine compare")
    # live FP64 peak: cuBLAS DGEMM on this box (MEASURED_PEAKS.json has no fp64 figure)
    d = 8192
    Xa = torch.randn(d, d, dtype=torch.float64, device=dev)
    Xb = torch.randn(d, d, dtype=torch.float64, device=dev)
    for _ in range(2):
        torch.matmul(Xa, Xb)
    best = 1e9
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(Xa, Xb)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    dgemm_peak = 2 * d ** 3 / best / 1e12
    del Xa, Xb

    chain = stats_acc.get("chain", [0, 0.0, 0.0])
    achieved = chain[2] / (chain[1] / 1e3) / 1e12 if chain[1] > 0 else None
    traffic, tinfo = load_traffic(nb, engine_used)
    if engine_used == "ozaki":
        npairs = args.oz_slices * (args.oz_slices + 1) // 2
        i8_peak, i8_how = int8_peak()
        roofline = {"bound": "tensor", "achieved": achieved * npairs if achieved else None, "peak": i8_peak,
                    "unit": "TOPS (int8)", "frac": achieved * npairs / i8_peak if achieved else None,
                    "traffic": traffic, "fp64_equivalent_tflops": achieved,
                    "kernel": "k_tc (persistent tensor-core kernel: all GEMM/SYRK tasks, FP64 tiles as "
                              f"{npairs} int8 tcgen05 GEMMs each (Ozaki I, s={args.oz_slices}))",
                    "achieved_how": "algorithmic GEMM/SYRK flops of k_tc (n^3/3 - Nt nb^3/3 - TRSM flops) x "
                                    f"{npairs} int8 products per FP64 multiply-add / its CUDA-event duration on "
                                    "its stream, summed over the timed steps",
                    "peak_how": i8_how,
                    "traffic_how": "dram__bytes_read.sum+dram__bytes_write.sum of one captured k_tc launch "
                                   "(profiles/ncu_tc_latest.json)" if traffic else None,
                    "fp64_dgemm_peak_live": None}
    roofline = roofline if engine_used == "ozaki" else {"bound": "tensor", "achieved": achieved, "peak": dgemm_peak, "unit": "TFLOP/s",
                "frac": achieved / dgemm_peak if achieved else None, "traffic": traffic,
                "kernel": "k_sched (persistent static-schedule kernel: FP64 DMMA GEMM/SYRK + TRSM tasks, "
                          "all flops but the diagonal POTRFs)",
                "achieved_how": "algorithmic flops of k_sched (n^3/3 - Nt*nb^3/3 per launch) / its CUDA-event "
                                "duration on its stream, summed over the timed steps",
                "peak_how": "cuBLAS DGEMM 8192^3 measured live in this run (fp64 dense; "
                            "MEASURED_PEAKS.json has no fp64 figure)",
                "traffic_how": "dram__bytes_read.sum+dram__bytes_write.sum of one captured k_sched launch "
                               "(profiles/ncu_chain_latest.json)" if traffic else None}
    if engine_used == "ozaki":
        roofline["fp64_dgemm_peak_live"] = dgemm_peak
    kstats = {k: {"launches": v[0], "ms": v[1], "tflops": (v[2] / (v[1] / 1e3) / 1e12) if v[1] > 0 and v[2] > 0
                  else None} for k, v in stats_acc.items()}

    progress("dgemm peak")
    # cuSOLVER potrf (cusolverDnXpotrf, fp64) on the same box (library baseline).
    # Its lower-triangle path dies with an illegal address at exactly n = 65536
    # (n^2 = 2^32; 65024 works), so it is timed lower at n - 512 (same family,
    # same lda layout) and upper at n (the other cuSOLVER code path).
    cusolver = None
    if not args.no_cusolver and ws == 1:
        from tools.cusolver_ref import Potrf
        cusolver = {}
        for label, nn, uplo in (("lower_n%d" % (n - 512 if n >= 65536 else n), n - 512 if n >= 65536 else n, 0),
                                ("upper_n%d" % n, n, 1)):
            Bv = B[:nn, :nn]
            ref = Potrf(nn, B.stride(1), Bv.data_ptr(), stream.cuda_stream, uplo)
            ts = []
            for i in range(2):
                B.copy_(A)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                ref(Bv.data_ptr())
                e1.record(stream)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) / 1e3)
            cinfo = int(ref.info.item())
            ref.close()
            cusolver[label] = {"value": nn ** 3 / 3 / min(ts) / 1e12, "unit": "TFLOP/s", "ms": min(ts) * 1e3,
                               "info": cinfo, "n": nn, "uplo": "L" if uplo == 0 else "U"}
        cusolver["note"] = ("cusolverDnXpotrf lower crashes (illegal address) at n=65536 exactly on CUDA 12.9 "
                            "(cuSOLVER 11.7.5); lower timed at n-512, upper at n; best of 2 each")
    del B
    plan.close()
    del plan
    torch.cuda.empty_cache()

    progress("cusolver")
    # end-to-end through the host API: pinned host A, H2D + factor + D2H per
    # step.  Several ranks: each rank streams (and writes back) only the tile
    # rows it owns from its own pinned copy of A.
    e2e = None
    if not args.no_e2e:
        torch.cuda.empty_cache()
        Ah = torch.empty((n, n), dtype=torch.float64).pin_memory()
        p2 = new_plan(n, nb)
        ts = []
        hb = db = 0
        for i in range(1 + args.e2e_steps):
            Ah.copy_(A.T)  # fresh input (row-major symmetric == column-major A), untimed
            torch.cuda.synchronize()
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(torch.cuda.current_stream())
            info = p2.factor(Ah.T)
            e1.record(torch.cuda.current_stream())
            torch.cuda.synchronize()
            assert info == 0, info
            if i >= 1:
                ts.append(e0.elapsed_time(e1) / 1e3)
            hb, db = p2.get("h2d_bytes"), p2.get("d2h_bytes")
        t = allreduce(sum(ts) / len(ts), "max")
        hb, db = int(allreduce(hb, "sum")), int(allreduce(db, "sum"))
        e2e = {"value": flops / t / 1e12, "unit": "TFLOP/s", "h2d_bytes_per_step": hb,
               "d2h_bytes_per_step": db, "ms_per_step": t * 1e3,
               "how": "mxp_chol_factor on a pinned host n x n matrix (per rank: its own tile rows); "
                      "CUDA events around the call, max over ranks"}
        p2.close()
        del Ah
    del A
    torch.cuda.empty_cache()

    progress("e2e")
    # C3 (BASELINE configs[2]): Matern nu=0.5 weak correlation, n = 131072, 4-precision maps
    # over eps in {1e-5 ... 1e-9}, tiles generated on the device inside the schedule.  FP64
    # references: our FP64 run and cuSOLVER potrf on the dense 137 GB matrix (independent).
    # Log-likelihood (Eq. 1) at y = 0 (Eq. 3 convention) and at y = Sigma z (z seeded normal), for
    # which y^T Sigma^-1 y = y^T z exactly (G16).
    mxp = None
    if not args.no_mxp:
        mxp = run_c3(args, m, dev, dev_index, stream, ws, new_plan, allreduce, barrier, dgemm_peak)

    progress("C3")
    kl = None
    if not args.no_kl and ws == 1:
        kl = run_kl_sweep(args, m, dev, new_plan)
        progress("KL sweep")
    # Out of core (a5/a9; C4's mode at a size this box's host RAM holds): the
    # host matrix streamed through HBM capped at ooc_frac of the lower
    # triangle vs the same host-streaming call with every tile resident, with
    # the C2 FP64 engine (Ozaki: fp64 ring + slice images recycled when their
    # row dies; DMMA: dead-tile slot recycling); plgsy FP64, nb as C2.  A third,
    # profiled out-of-core run records the per-column C2G / G2C / Work timeline.
    ooc = None
    if not args.no_ooc and ws == 1:
        import gc
        no, nbo = args.ooc_n, args.nb
        nto = -(-no // nbo)
        lower = nto * (nto + 1) // 2 * nbo * nbo * 8
        gc.collect()
        torch.cuda.empty_cache()
        Ah = torch.empty((no, no), dtype=torch.float64).pin_memory()

        def fresh():
            Ad = torch.empty((no, no), dtype=torch.float64, device=dev).T
            m.generate_plgsy_device(Ad, seed=args.seed, stream=stream.cuda_stream)
            Ah.copy_(Ad.T)
            del Ad
            torch.cuda.synchronize()
            torch.cuda.empty_cache()

        def run_ooc(cap, profile=False):
            ts, hb, db, slots, extra = [], 0, 0, 0, {}
            for i in range(1 if profile else 2):  # first call: warm-up (plan workspace, pinned stage)
                fresh()
                pl = m.Plan(no, nbo)
                pl.set("device", dev_index)
                pl.set("fp64_engine", ENG[args.fp64_engine])
                pl.set("oz_slices", args.oz_slices)
                if cap:
                    pl.set("hbm_bytes_cap", cap)
                if profile:
                    pl.set("profile", 1)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                inf = pl.factor(Ah.T)
                e1.record(stream)
                torch.cuda.synchronize()
                assert inf == 0, inf
                ts.append(e0.elapsed_time(e1) / 1e3)
                hb, db, slots = pl.get("h2d_bytes"), pl.get("d2h_bytes"), pl.get("pool_slots")
                extra = {"fp64_engine": "ozaki" if pl.get("fp64_engine_used") == 1 else "dmma",
                         "oz_image_slots": pl.get("oz_image_slots")}
                if profile:
                    extra["timeline"] = pl.timeline()
                pl.close()
                del pl
                gc.collect()
                torch.cuda.empty_cache()
            return ts[-1], hb, db, slots, extra

        t_in, hb_in, db_in, s_in, x_in = run_ooc(0)
        cap = int(args.ooc_frac * lower)
        t_oc, hb_oc, db_oc, s_oc, x_oc = run_ooc(cap)
        t_pr, _, _, _, x_pr = run_ooc(cap, profile=True)
        fl = no ** 3 / 3
        ooc = {"workload": f"plgsy n={no} nb={nbo} FP64 from pinned host memory (mxp_chol_factor)",
               "lower_triangle_gb": round(lower / 1e9, 2),
               "in_core": dict({"tflops": fl / t_in / 1e12, "ms": t_in * 1e3, "pool_slots": s_in,
                                "h2d_bytes": hb_in, "d2h_bytes": db_in}, **x_in),
               "out_of_core": dict({"tflops": fl / t_oc / 1e12, "ms": t_oc * 1e3, "pool_slots": s_oc,
                                    "hbm_cap_gb": round(cap / 1e9, 2), "h2d_bytes": hb_oc, "d2h_bytes": db_oc},
                                   **x_oc),
               "ooc_over_in_core": t_in / t_oc,
               "ooc_over_c2_device_in_core": (fl / t_oc / 1e12) / value,
               "variants": ooc_variant_ledgers(m, no, nbo, lower, [args.ooc_frac, 0.35], hb_oc, db_oc),
               "timeline": ooc_timeline_summary(x_pr.get("timeline"), t_pr),
               "note": "C4 (n=262144, 276 GB lower triangle) exceeds this box's 196 GB host RAM; the same "
                       "streaming/recycling path is timed with the pool capped below the lower triangle"}
        del Ah
        gc.collect()

    cpu = None
    cpu_table = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        cpu = cpu_oracle_sample(2048, 256, args.seed)
        cpu.pop("seconds", None)
        try:
            cpu_table = cpu_baselines(args.seed)
        except Exception as e:  # noqa
            cpu_table = {"error": repr(e)[:200]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": "f64" if engine_used == "dmma" else "f64 (Ozaki-I: int8 tcgen05 slice products, int32/fp64 accumulation)",
            "data": "synthetic",
            "config": {"workload": f"C2: plgsy random SPD n={n} nb={nb} FP64 in-core on B200, "
                                   f"device-resident input", "n": n, "nb": nb, "seed": args.seed,
                       "fp64_engine": engine_used,
                       "l2": "inputs (n^2*8 B = %.1f GB) larger than L2 (126 MB); no flush" % (n * n * 8 / 1e9),
                       "parallelism": "single GPU" if ws == 1 else
                       f"row-cyclic over {ws} ranks (tile row m on rank m mod {ws}); finished tiles pushed "
                       f"peer-to-peer by the copy engines" + (" [ranks co-located on one GPU, SM-partitioned: "
                                                             "a functional run, not a scaling number]" if coloc else "")},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "clocks": ck,
            "baselines": {"cusolver_potrf": cusolver, "cpu": cpu_table},
            "mxp_c3": mxp,
            "kl_sweep": kl,
            "ooc": ooc,
            "sched": sched,
            "check": {"backward_error_fro": backward_error, "backward_error_probe": probe, "logdet": logdet,
                      "how": "||A - L L^T||_F / ||A||_F by block columns of cuBLAS DGEMM (bar 1e-13, north_star); "
                             "probe = ||(A - L L^T) x|| / ||A x||, x: 4 seeded normal columns"},
            "fp64_engines": engines,
            "kernels": kstats,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
