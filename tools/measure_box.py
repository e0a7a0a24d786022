"""Measure the B200 box facts DESIGN.md's rooflines need (run under gpurun).

DGEMM (cuBLAS via torch.matmul fp64), cuSOLVER potrf (torch.linalg.cholesky),
TF32/FP16/FP8 matmul peaks, pinned H2D/D2H bandwidth, host cores and RAM.
Writes gpurun_out/box_facts.json.
"""
import json, os, subprocess, time
import torch

out = {}
out["nproc"] = os.cpu_count()
try:
    out["free_g"] = subprocess.run(["free", "-g"], capture_output=True, text=True).stdout
    out["lscpu"] = subprocess.run(["lscpu"], capture_output=True, text=True).stdout[:3000]
    out["numa"] = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout
except Exception as e:  # noqa
    out["err"] = str(e)
dev = torch.device("cuda:0")
out["gpu"] = torch.cuda.get_device_name(0)


def timeit(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) / 1e3)
    return min(ts), sorted(ts)[len(ts) // 2]


for n in (8192, 16384):
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    tmin, tmed = timeit(lambda: torch.matmul(a, b))
    out[f"dgemm_{n}_tflops_best"] = 2 * n**3 / tmin / 1e12
    out[f"dgemm_{n}_tflops_med"] = 2 * n**3 / tmed / 1e12
    del a, b
# dgemm with nb=1024 inner shape typical of the left-looking update: M=32768, N=1024, K=32768
a = torch.randn(32768, 32768, dtype=torch.float64, device=dev)
b = torch.randn(1024, 32768, dtype=torch.float64, device=dev)
tmin, tmed = timeit(lambda: torch.matmul(a, b.t()))
out["dgemm_M32768_N1024_K32768_tflops_best"] = 2 * 32768 * 1024 * 32768 / tmin / 1e12
del a, b
torch.backends.cuda.matmul.allow_tf32 = True
for dt, name in ((torch.float32, "tf32"), (torch.float16, "fp16")):
    n = 8192
    a = torch.randn(n, n, dtype=dt, device=dev); b = torch.randn(n, n, dtype=dt, device=dev)
    tmin, _ = timeit(lambda: torch.matmul(a, b), reps=10)
    out[f"{name}_8192_tflops_best"] = 2 * n**3 / tmin / 1e12
torch.backends.cuda.matmul.allow_tf32 = False
n = 8192
a = torch.randn(n, n, dtype=torch.float32, device=dev); b = torch.randn(n, n, dtype=torch.float32, device=dev)
tmin, _ = timeit(lambda: torch.matmul(a, b), reps=5)
out["sgemm_8192_tflops_best"] = 2 * n**3 / tmin / 1e12
try:
    a8 = torch.randn(n, n, device=dev).to(torch.float8_e4m3fn)
    b8 = torch.randn(n, n, device=dev).to(torch.float8_e4m3fn)
    one = torch.tensor(1.0, device=dev)
    tmin, _ = timeit(lambda: torch._scaled_mm(a8, b8.t(), scale_a=one, scale_b=one, out_dtype=torch.bfloat16), reps=10)
    out["fp8_8192_tflops_best"] = 2 * n**3 / tmin / 1e12
except Exception as e:
    out["fp8_err"] = str(e)[:200]
del a, b
torch.cuda.empty_cache()

# cuSOLVER potrf via torch.linalg.cholesky
def spd(n):
    g = torch.Generator(device=dev); g.manual_seed(42)
    A = torch.rand(n, n, dtype=torch.float64, device=dev, generator=g) - 0.5
    A = (A + A.t()) * 0.5
    A.diagonal().add_(n)
    return A
for n in (16384, 32768, 65536):
    A = spd(n)
    def f():
        return torch.linalg.cholesky_ex(A, upper=False)
    reps = 3 if n >= 65536 else 5
    tmin, tmed = timeit(f, reps=reps, warm=1)
    out[f"cusolver_potrf_{n}_tflops_best"] = n**3 / 3 / tmin / 1e12
    out[f"cusolver_potrf_{n}_tflops_med"] = n**3 / 3 / tmed / 1e12
    del A
    torch.cuda.empty_cache()

# pinned H2D / D2H
nbytes = 4 << 30
h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
tmin, _ = timeit(lambda: d.copy_(h, non_blocking=True), reps=5)
out["h2d_pinned_GBps"] = nbytes / tmin / 1e9
tmin, _ = timeit(lambda: h.copy_(d, non_blocking=True), reps=5)
out["d2h_pinned_GBps"] = nbytes / tmin / 1e9
s2 = torch.cuda.Stream()
def both():
    with torch.cuda.stream(s2):
        h[: nbytes // 2].copy_(d[: nbytes // 2], non_blocking=True)
    d[nbytes // 2:].copy_(h[nbytes // 2:], non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)
tmin, _ = timeit(both, reps=5)
out["bidir_pinned_GBps_total"] = nbytes / tmin / 1e9
t0 = time.time(); hh = torch.empty(16 << 30, dtype=torch.uint8, pin_memory=True); out["pin_alloc_16GiB_s"] = time.time() - t0
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/box_facts.json", "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if not isinstance(v, str)}, indent=1))
