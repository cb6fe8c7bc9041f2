"""N>1 path on CPU: the row-sharded boundary-graph Floyd-Warshall protocol of
engine_fw.cuh:run_fw_sharded, modelled in numpy and run as world_size-2/3
`gloo` processes. The CUDA kernels are the single-GPU ones; what this pins is
the ownership and exchange logic:

* owner(I) = I mod world; panel slot J comes from the owner of its home row
  (kb for J > kb, J for J < kb); phase 3 touches owned upper tiles only;
* the sparse walk: phase 2 marks a slot active iff it holds a finite entry
  (an all-INF slot stays all-INF), phase 3 walks only active x active tiles;
* exchange "p2p" (the default on GPUs): the diagonal tile comes from its
  owner, then every rank pulls from each slot's owner the activity flag and,
  only for active slots, the tile (modelled by all_gather_object of the
  owned active slots); exchange "allreduce" (PSP_K2_EXCHANGE=nccl): non-owned
  slots are INF and flagged inactive, one min-allreduce of tiles and flags;
* the K2 elimination order: the matrix is closed in a permuted numbering and
  permuted back, which must not change a single entry;
* row-sharded storage (PSP_STORAGE_ROW_SHARDED): rows a rank does not own
  hold garbage (NaN here, the sink allocation on GPUs) and must never be
  read -- the diagonal tile of a foreign k-block goes to a scratch tile --,
  there is no replication, and each destination's boundary rows are
  assembled by a min-reduce of every rank's part (engine_shard.cuh
  gather_bt_part + ncclReduce).
"""
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


def sharded_fw(D: np.ndarray, rank: int, world: int, dist, mode: str = "p2p",
               perm: np.ndarray | None = None, rows_only: bool = False) -> tuple[np.ndarray, int]:
    """Returns the closed matrix (original numbering) and the number of bytes
    of panel tiles this rank received. rows_only: row-sharded storage; the
    result then holds only the rows t with t % world == rank (others NaN),
    gathered from every rank's owned tile rows."""
    import torch
    n = D.shape[0]
    if perm is not None:  # position perm[i] holds vertex i
        P = np.empty_like(D)
        P[np.ix_(perm, perm)] = D
        D = P
    nb = -(-n // T)
    N = nb * T
    M = np.full((N, N), np.inf)
    M[:n, :n] = D
    np.fill_diagonal(M, 0.0)
    tile = lambda I, J: (slice(I * T, (I + 1) * T), slice(J * T, (J + 1) * T))
    if rows_only:  # rows of other ranks are not stored: garbage that must never be read
        for I in range(nb):
            if I % world != rank:
                M[I * T:(I + 1) * T, :] = np.nan
    received = 0
    for kb in range(nb):
        owner = kb % world
        K = tile(kb, kb)
        if rank == owner:  # phase 1 on the diagonal tile
            d = M[K]
            for k in range(T):
                d = np.minimum(d, d[:, k:k + 1] + d[k:k + 1, :])
            M[K] = d
        t = torch.from_numpy(np.ascontiguousarray(M[K]))
        dist.broadcast(t, src=owner)  # p2p: pull_diag from the owner's region
        if rows_only and rank != owner:
            dkk = t.numpy().copy()  # MatSet::diag scratch tile
        else:
            M[K] = t.numpy()
            dkk = M[K]
        # phase 2 on owned slots: slot J = D[kb rows][J cols]; flag 0 = active
        panel = np.full((nb, T, T), np.inf)
        flag = np.ones(nb, np.int8)
        mine = {}
        for J in range(nb):
            if J == kb:
                continue
            home = kb if J > kb else J
            if home % world != rank:
                continue
            R = M[tile(kb, J)] if J > kb else M[tile(J, kb)].T
            if not np.isfinite(R).any():
                flag[J] = 1  # all INF stays all INF: not computed
                mine[J] = None
                continue
            R = np.min(dkk[:, :, None] + R[None, :, :], axis=1)
            assert np.isfinite(R).any()
            panel[J], flag[J] = R, 0
            mine[J] = R
            if J > kb:
                M[tile(kb, J)] = R
            else:
                M[tile(J, kb)] = R.T
        if mode == "p2p":
            # every rank reads each owner's flags and pulls the active tiles
            pubs = [None] * world
            dist.all_gather_object(pubs, mine)
            for r, pub in enumerate(pubs):
                if r == rank:
                    continue
                for J, R in pub.items():
                    if R is None:
                        flag[J] = 1
                    else:
                        panel[J], flag[J] = R, 0
                        received += R.nbytes
        else:
            pt = torch.from_numpy(panel)
            ft = torch.from_numpy(flag.astype(np.float64))
            dist.all_reduce(pt, op=dist.ReduceOp.MIN)
            dist.all_reduce(ft, op=dist.ReduceOp.MIN)
            panel, flag = pt.numpy(), ft.numpy().astype(np.int8)
            received += panel.nbytes
        active = [J for J in range(nb) if J != kb and flag[J] == 0]
        # phase 3: owned rows, upper tiles, active x active only
        for I in active:
            if I % world != rank:
                continue
            for J in active:
                if J < I:
                    continue
                A, B = panel[I], panel[J]          # A[k][i] = D[i][k] by symmetry
                M[tile(I, J)] = np.minimum(M[tile(I, J)],
                                           np.min(A[:, :, None] + B[:, None, :], axis=0))
    if rows_only:
        # gather_bt_part: destination d's rows (here t % world == d), each
        # element from the rank holding its tile row min(p, q) / T, INF from
        # the others; min-reduced at d
        pos = perm if perm is not None else np.arange(n)
        mine_rows = None
        for d in range(world):
            rows = np.arange(d, n, world)
            part = np.full((len(rows), n), np.inf)
            for a, t in enumerate(rows):
                p = pos[t]
                for j in range(n):
                    q = pos[j]
                    if (min(p, q) // T) % world == rank:
                        part[a, j] = M[min(p, q), max(p, q)] if p // T <= q // T else M[q, p]
            pt = torch.from_numpy(part)
            dist.reduce(pt, dst=d, op=dist.ReduceOp.MIN)
            if d == rank:
                mine_rows = (rows, pt.numpy())
        out = np.full((n, n), np.nan)
        out[mine_rows[0]] = mine_rows[1]
        return out, received
    for I in range(nb):  # replicate rows from their owners
        rowt = torch.from_numpy(np.ascontiguousarray(M[I * T:(I + 1) * T, I * T:]))
        dist.broadcast(rowt, src=I % world)
        M[I * T:(I + 1) * T, I * T:] = rowt.numpy()
    full = M.copy()
    for I in range(nb):
        for J in range(I):
            full[tile(I, J)] = M[tile(J, I)].T
    full = full[:n, :n]
    if perm is not None:
        full = full[np.ix_(perm, perm)]
    return full, received


def _worker(rank, world, port, D, mode, perm, out_q, rows_only=False):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = sharded_fw(D, rank, world, dist, mode, perm, rows_only)
    out_q.put((rank, res))
    dist.barrier()
    dist.destroy_process_group()


def _two_pieces():
    """Two disconnected triangulated grids: panel slots of one piece stay all
    INF against the other, so the sparse walk and the flags matter."""
    import paper_1503_07192_b200 as P
    a = P.generate_triangulated_grid(4, 5, (1.0, 9.0), 3)
    b = P.generate_triangulated_grid(3, 6, (1.0, 9.0), 4)
    n = a.n + b.n
    eu = np.concatenate([a.eu, b.eu + a.n])
    ev = np.concatenate([a.ev, b.ev + a.n])
    ew = np.concatenate([a.ew, b.ew])
    return n, eu, ev, ew


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("mode", ["p2p", "allreduce"])
@pytest.mark.parametrize("case", ["grid", "two_pieces_permuted"])
def test_row_sharded_fw_protocol_gloo(world, mode, case):
    import torch.multiprocessing as mp
    import paper_1503_07192_b200 as P
    if case == "grid":
        g = P.generate_triangulated_grid(5, 8, (1.0, 9.0), 3)
        n, eu, ev, ew = g.n, g.eu, g.ev, g.ew
        perm = None
    else:
        n, eu, ev, ew = _two_pieces()
        # interleave the pieces (an elimination order that is not the natural one)
        perm = np.random.default_rng(5).permutation(n)
    D = np.full((n, n), np.inf)
    D[eu, ev] = ew
    D[ev, eu] = ew
    np.fill_diagonal(D, 0)
    truth = oracle.apsp_dense(n, eu, ev, ew)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, D, mode, perm, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert np.array_equal(results[r][0], truth), f"rank {r}"
    if mode == "p2p" and case == "two_pieces_permuted":
        # only active slots move: less than the all-reduce's full panels
        nb = -(-n // T)
        assert sum(results[r][1] for r in range(world)) < world * nb * nb * T * T * 8


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("mode", ["p2p", "allreduce"])
def test_row_sharded_storage_protocol_gloo(world, mode):
    # no rank reads a row it does not own (NaN would spread), and the
    # min-reduce gather gives every destination its exact rows
    import torch.multiprocessing as mp
    n, eu, ev, ew = _two_pieces()
    perm = np.random.default_rng(7).permutation(n)
    D = np.full((n, n), np.inf)
    D[eu, ev] = ew
    D[ev, eu] = ew
    np.fill_diagonal(D, 0)
    truth = oracle.apsp_dense(n, eu, ev, ew)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, D, mode, perm, q, True))
             for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        rows = np.arange(r, n, world)
        got = results[r][0][rows]
        assert not np.isnan(got).any(), f"rank {r} read a row it does not own"
        assert np.array_equal(got, truth[rows]), f"rank {r}"
