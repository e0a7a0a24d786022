"""CPU (gloo, world_size 2) checks of the multi-GPU host logic: the per-rank
static task lists partition the single-rank list exactly (row-cyclic owner
map); no GPU work is issued."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, nb, pmap, q):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import __graft_entry__
    __graft_entry__.build()
    import paper_2410_09819_b200 as m
    res = {}
    for streaming in (False, True):
        plan = m.Plan(n, nb, pmap)
        plan.set("rank", rank)
        plan.set("nranks", world)
        c = plan.describe(streaming)
        t = torch.tensor([c[k] for k in sorted(c)], dtype=torch.int64)
        dist.all_reduce(t)
        res[streaming] = dict(zip(sorted(c), t.tolist()))
        mine = torch.tensor([c["owned_tiles"]], dtype=torch.int64)
        got = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(got, mine)
        res[(streaming, "owned")] = [int(x) for x in got]
    if rank == 0:
        q.put(res)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_rank_lists_partition_the_schedule(world):
    import oracle
    import paper_2410_09819_b200 as m
    import workloads as w
    n, nb = 4096, 256
    xy = w.matern_locations(n, seed=1)
    pmap = oracle.plan(w.matern_cov(xy, 1.0, 0.02627), nb, 1e-5)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, nb, pmap, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for streaming in (False, True):
        single = m.Plan(n, nb, pmap).describe(streaming)
        assert res[streaming] == single, (streaming, res[streaming], single)
        Nt = n // nb
        owned = res[(streaming, "owned")]
        assert sum(owned) == Nt * (Nt + 1) // 2
        assert max(owned) - min(owned) <= Nt  # row-cyclic balance
