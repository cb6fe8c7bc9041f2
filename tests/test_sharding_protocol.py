"""N>1 path on CPU: the row-sharded boundary-graph Floyd-Warshall protocol of
psp_gpu.cu:run_fw_sharded, modelled in numpy and run as world_size-2 `gloo`
processes with the same collectives (diagonal-tile broadcast, panel
min-allreduce, final per-row broadcast). The CUDA kernels are the
single-GPU ones; what this pins is the ownership and exchange logic:
owner(I) = I mod world, panel tile J comes from the owner of its home row
(kb for J > kb, J for J < kb), phase 3 touches owned upper tiles only."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

import oracle

T = 4  # small tile so a 40-vertex graph spans 10 tile rows


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def sharded_fw(D: np.ndarray, rank: int, world: int, dist) -> np.ndarray:
    import torch
    n = D.shape[0]
    nb = -(-n // T)
    N = nb * T
    M = np.full((N, N), np.inf)
    M[:n, :n] = D
    np.fill_diagonal(M, 0.0)
    tile = lambda I, J: (slice(I * T, (I + 1) * T), slice(J * T, (J + 1) * T))
    for kb in range(nb):
        owner = kb % world
        K = tile(kb, kb)
        if rank == owner:  # phase 1 on the diagonal tile
            d = M[K]
            for k in range(T):
                d = np.minimum(d, d[:, k:k + 1] + d[k:k + 1, :])
            M[K] = d
        t = torch.from_numpy(np.ascontiguousarray(M[K]))
        dist.broadcast(t, src=owner)
        M[K] = t.numpy()
        dkk = M[K]
        # phase 2: panel slot J = R_J = D[kb rows][J cols], from its home row
        panel = np.full((nb, T, T), np.inf)
        for J in range(nb):
            if J == kb:
                continue
            home = kb if J > kb else J
            if home % world != rank:
                continue
            R = M[tile(kb, J)] if J > kb else M[tile(J, kb)].T
            R = np.min(dkk[:, :, None] + R[None, :, :], axis=1)
            panel[J] = R
            if J > kb:
                M[tile(kb, J)] = R
            else:
                M[tile(J, kb)] = R.T
        pt = torch.from_numpy(panel)
        dist.all_reduce(pt, op=dist.ReduceOp.MIN)
        panel = pt.numpy()
        # phase 3 on owned rows, upper tiles only
        for I in range(rank, nb, world):
            for J in range(I, nb):
                if I == kb or J == kb:
                    continue
                A, B = panel[I], panel[J]          # A[k][i] = D[i][k] by symmetry
                M[tile(I, J)] = np.minimum(M[tile(I, J)],
                                           np.min(A[:, :, None] + B[:, None, :], axis=0))
    for I in range(nb):  # replicate rows from their owners
        rowt = torch.from_numpy(np.ascontiguousarray(M[I * T:(I + 1) * T, I * T:]))
        dist.broadcast(rowt, src=I % world)
        M[I * T:(I + 1) * T, I * T:] = rowt.numpy()
    U = np.triu(np.ones((nb, nb), bool))
    full = M.copy()
    for I in range(nb):
        for J in range(I):
            full[tile(I, J)] = M[tile(J, I)].T
    assert U.any()
    return full[:n, :n]


def _worker(rank, world, port, D, out_q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = sharded_fw(D, rank, world, dist)
    out_q.put((rank, res))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_row_sharded_fw_protocol_gloo(world):
    import torch.multiprocessing as mp
    import paper_1503_07192_b200 as P
    g = P.generate_triangulated_grid(5, 8, (1.0, 9.0), 3)
    D = np.full((g.n, g.n), np.inf)
    D[g.eu, g.ev] = g.ew
    D[g.ev, g.eu] = g.ew
    np.fill_diagonal(D, 0)
    truth = oracle.apsp_dense(g.n, g.eu, g.ev, g.ew)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, D, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert np.array_equal(results[r], truth), f"rank {r}"
