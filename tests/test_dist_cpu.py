"""Multi-process host logic of the multi-GPU path on CPU (gloo, world_size 2): eigenpair
range partition and the column gather reproduce the single-process result exactly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1912_04062_b200.dist import eigpair_range, gather_columns


def test_eigpair_range_partition():
    for nev in [1, 7, 64, 16384]:
        for world in [1, 2, 3, 4, 8]:
            if world > nev:
                continue
            rngs = [eigpair_range(nev, r, world) for r in range(world)]
            assert rngs[0][0] == 0 and rngs[-1][1] == nev
            assert all(rngs[i][1] == rngs[i + 1][0] for i in range(world - 1))
            sizes = [k1 - k0 for k0, k1 in rngs]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, nev, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import skewgen
    A = skewgen.random_skew(n, n)
    lam, Zre, Zim, st = oracle.skew_eig(A, nev)   # stands in for the per-rank CUDA solve
    k0, k1 = eigpair_range(nev, rank, world)
    full_re = gather_columns(torch.from_numpy(np.ascontiguousarray(Zre[:, k0:k1])), nev)
    full_im = gather_columns(torch.from_numpy(np.ascontiguousarray(Zim[:, k0:k1])), nev)
    if rank == 0:
        out["ok"] = bool(np.array_equal(full_re.numpy(), Zre) and np.array_equal(full_im.numpy(), Zim))
    dist.barrier()
    dist.destroy_process_group()


def test_gather_columns_world2_gloo():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), 40, 19, out), nprocs=2, join=True)
    assert out.get("ok") is True
