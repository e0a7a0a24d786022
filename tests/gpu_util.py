"""Helpers for the -m gpu parity tests: run the CUDA path through the C ABI."""
import numpy as np


def gpu_factor(A, nb, pmap=None, attrs=None, host=False, plan=None):
    import torch

    import paper_2410_09819_b200 as m
    n = A.shape[0]
    if plan is None:
        plan = m.Plan(n, nb, pmap)
    for k, v in (attrs or {}).items():
        plan.set(k, v)
    if host:
        Ah = torch.tensor(np.asfortranarray(A)).T.contiguous().T  # column-major CPU tensor
        info = plan.factor(Ah)
        L = np.tril(Ah.numpy())
    else:
        Ad = torch.tensor(np.ascontiguousarray(A.T), device="cuda").T  # column-major view of A
        info = plan.factor_device(Ad)
        torch.cuda.synchronize()
        L = np.tril(Ad.cpu().numpy())
    ld = plan.logdet() if info == 0 else None
    return L, info, ld, plan
