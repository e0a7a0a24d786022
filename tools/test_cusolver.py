import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_09819_b200 as m
from tools.cusolver_ref import Potrf
uplo = int(os.environ.get('UPLO', '0'))
for n in [int(x) for x in sys.argv[1:]]:
    A = torch.empty((n, n), dtype=torch.float64, device="cuda").T
    m.generate_plgsy_device(A, 42)
    B = A.clone(memory_format=torch.contiguous_format).T.contiguous().T if False else torch.empty((n, n), dtype=torch.float64, device="cuda").T
    B.copy_(A)
    torch.cuda.synchronize()
    ref = Potrf(n, B.stride(1), B.data_ptr(), torch.cuda.current_stream().cuda_stream, uplo)
    print(n, "ws bytes", ref.dws, ref.hws, flush=True)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); ref(B.data_ptr()); e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3
    L = torch.tril(B) if uplo == 0 else torch.triu(B).T
    x = torch.randn(n, 2, dtype=torch.float64, device="cuda")
    r = ((A @ x - L @ (L.T @ x)).norm() / (torch.linalg.matrix_norm(A) * x.norm())).item()
    print(f"n={n} info={ref.info.item()} t={t:.3f} {n**3/3/t/1e12:.2f} TF probe={r:.2e}", flush=True)
    ref.close(); del A, B, L; torch.cuda.empty_cache()
