"""cuSOLVER FP64 reference for C3 (run by bench.py in its own process: a cuSOLVER fault must
not take the bench's CUDA context down).  Library baseline only -- none of our kernels
factor anything here; the Matern covariance comes from the repo's device generator.

    python tools/cusolver_c3.py n range_a out.npz

Writes logdet, y^T Sigma^-1 y (cusolverDnXpotrs), the exact z^T Sigma z, timing and y = Sigma z
(z: seeded standard normal, seed 2) for the caller's log-likelihood checks.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch

    import paper_2410_09819_b200 as m
    import workloads as w
    from tools.cusolver_ref import Potrf, potrs
    n, a, out = int(sys.argv[1]), float(sys.argv[2]), sys.argv[3]
    dev = torch.device("cuda", 0)
    xyd = torch.as_tensor(w.matern_locations(n, seed=1), device=dev).contiguous()
    z = torch.randn(n, dtype=torch.float64, device=dev, generator=torch.Generator(device=dev).manual_seed(2))
    A = torch.empty((n, n), dtype=torch.float64, device=dev).T
    stream = torch.cuda.current_stream()
    m.generate_matern_device(A, xyd, 1.0, a, stream=stream.cuda_stream)
    y = A @ z
    q_exact = float(y @ z)
    ref = Potrf(n, A.stride(1), A.data_ptr(), stream.cuda_stream, 1)  # upper (lower faults at large n)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    ref(A.data_ptr())
    e1.record(stream)
    torch.cuda.synchronize()
    info = int(ref.info.item())
    logdet = 2.0 * torch.log(torch.diagonal(A)).sum().item()
    x = y.clone().unsqueeze(1)
    potrs(ref, A.data_ptr(), x.data_ptr())
    torch.cuda.synchronize()
    q = float(y @ x[:, 0])
    ref.close()
    ms = e0.elapsed_time(e1)
    np.savez(out, y=y.cpu().numpy(), meta=json.dumps({"n": n, "info": info, "logdet": logdet, "quad_form": q,
                                                      "quad_form_exact": q_exact, "ms": ms,
                                                      "tflops": n ** 3 / 3 / (ms / 1e3) / 1e12}))


if __name__ == "__main__":
    main()
