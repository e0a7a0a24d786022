import sys, os, time
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2410_09819_b200 as m
n, nb = int(sys.argv[1]), int(sys.argv[2])
frac = float(sys.argv[3])
Ad = torch.empty((n, n), dtype=torch.float64, device="cuda").T
m.generate_plgsy_device(Ad, seed=42, stream=torch.cuda.current_stream().cuda_stream)
Ah = torch.empty((n, n), dtype=torch.float64).pin_memory()
Ah.copy_(Ad.T); torch.cuda.synchronize(); print("host ready", flush=True)
del Ad; torch.cuda.empty_cache()
nt = -(-n // nb); lower = nt * (nt + 1) // 2 * nb * nb * 8
pl = m.Plan(n, nb)
if len(sys.argv) > 4: pl.set("device", 0)
if frac > 0: pl.set("hbm_bytes_cap", int(frac * lower))
print("slots", pl.get("pool_slots"), "T", nt * (nt + 1) // 2, flush=True)
t0 = time.time()
info = pl.factor(Ah.T)
torch.cuda.synchronize()
print("info", info, "s", time.time() - t0, flush=True)
