"""CPU (gloo, world_size 2 and 3) tests of the domain-decomposition communication layer.

The kernels are CUDA-only, so the multi-process path is covered here at the level it
adds to the single-GPU code: halo exchange of contiguous x-slabs, the fp64 L1 /
production all-reduce and the coarse-level all-gather, plus the slab layout rules.
"""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2301_09991_b200.dd import (GX, TorchDistComm, _edges, distributed_levels,
                                      slab_bounds)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, size, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        comm = TorchDistComm()
        nx, hx, w = 6, 4, 3
        # slab rows: interior value = 100 * rank + local x, ghosts start at -1
        t = torch.full((nx + 2 * hx, 5, 2), -1.0, dtype=torch.float64)
        for x in range(nx):
            t[hx + x] = 100.0 * rank + x
        comm.exchange(t, w, hx)
        we, ee, wg, eg = _edges(t, w, hx)
        ok = True
        if rank > 0:       # west ghost = west neighbour's east interior edge
            ok &= bool(torch.all(wg[:, 0, 0] == torch.tensor([100.0 * (rank - 1) + x
                                                              for x in range(nx - w, nx)],
                                                             dtype=torch.float64)))
        else:
            ok &= bool(torch.all(wg == -1.0))
        if rank < size - 1:
            ok &= bool(torch.all(eg[:, 0, 0] == torch.tensor([100.0 * (rank + 1) + x
                                                              for x in range(w)],
                                                             dtype=torch.float64)))
        else:
            ok &= bool(torch.all(eg == -1.0))
        # several fields in one grouped exchange (different widths / halos / shapes),
        # waited on after unrelated work
        fields = []
        for k, (n, h, ww) in enumerate(((8, 5, 3), (4, 5, 2), (6, 3, 1))):
            f = torch.full((n + 2 * h, 3), -1.0, dtype=torch.float64)
            for x in range(n):
                f[h + x] = 1000.0 * k + 100.0 * rank + x
            fields.append((f, ww, h, n, k))
        handle = comm.exchange_many([(f, ww, h) for f, ww, h, _, _ in fields])
        _ = torch.ones(4).sum()
        handle.wait()
        for f, ww, h, n, k in fields:
            _, _, wg2, eg2 = _edges(f, ww, h)
            if rank > 0:
                ok &= bool(torch.all(wg2[:, 0] == torch.tensor(
                    [1000.0 * k + 100.0 * (rank - 1) + x for x in range(n - ww, n)],
                    dtype=torch.float64)))
            else:
                ok &= bool(torch.all(wg2 == -1.0))
            if rank < size - 1:
                ok &= bool(torch.all(eg2[:, 0] == torch.tensor(
                    [1000.0 * k + 100.0 * (rank + 1) + x for x in range(ww)],
                    dtype=torch.float64)))
            else:
                ok &= bool(torch.all(eg2 == -1.0))
            # ghost rows beyond the exchanged width stay untouched
            ok &= bool(torch.all(f[:h - ww] == -1.0)) and bool(torch.all(f[h + n + ww:] == -1.0))
        l1 = torch.tensor([1.5 + rank], dtype=torch.float64)
        comm.allreduce_sum_(l1)
        ok &= abs(float(l1) - sum(1.5 + r for r in range(size))) < 1e-15
        g = comm.allgather_x(torch.full((2, 3), float(rank)))
        ok &= g.shape == (2 * size, 3) and all(float(g[2 * r, 0]) == r for r in range(size))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("size", [2, 3])
def test_gloo_halo_exchange_and_collectives(size):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, size, port, q)) for r in range(size)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    results = dict(q.get(timeout=5) for _ in range(size))
    assert all(results[r] for r in range(size)), results
    assert all(p.exitcode == 0 for p in procs)


def test_slab_layout_rules():
    assert slab_bounds(512, 8, 3) == (192, 256)
    with pytest.raises(ValueError):
        slab_bounds(100, 8, 0)
    # C4 at 8 ranks: 64-column slabs stay distributed while >= 2 GX columns remain
    lg = distributed_levels(512, 512, 8, 10)
    assert (512 // 8) >> (lg - 1) >= 2 * GX and ((512 // 8) >> lg < 2 * GX or lg == 9)
    assert distributed_levels(64, 64, 4, 7) >= 1
