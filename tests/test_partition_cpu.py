"""Host logic of the general-sparse row partition (kpm_csr_partition, include/kpm.h; SURVEY.md
8(f) NEXT-4) without a GPU: the ghost / send lists every rank derives on its own from the whole
matrix must fit together, and a world-size-2 gloo run that exchanges ghost values with exactly
those lists and applies the local rows (extended-block numbering) must reproduce H x."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import kpm_inputs as ki
import oracle


def sparse_cases():
    rng = np.random.default_rng(7)
    D = 61
    A = np.zeros((D, D))
    for i in range(D):
        for j in rng.choice(D, size=int(rng.integers(1, 5)), replace=False):
            A[i, j] += rng.normal()
    A = A + A.T
    lat = dict(ndim=3, L=(5, 4, 6), D=120, t=-1.0, onsite=ki.anderson_onsite(3, 120, 1.0), flux=0.0)
    return {"random": oracle.csr_from_dense(A), "lattice3d": oracle.lattice_csr(lat)}


def block_bounds(D, world):
    return [D * q // world for q in range(world + 1)]


@pytest.mark.parametrize("world", [1, 2, 3, 5])
@pytest.mark.parametrize("case", ["random", "lattice3d"])
def test_partition_lists_fit_together(case, world):
    from paper_1105_5481_b200 import kpm
    H = sparse_cases()[case]
    bnd = block_bounds(H.D, world)
    plans = [kpm.kpm_csr_partition(H.D, H.rowptr, H.col, g, world) for g in range(world)]
    for g, P in enumerate(plans):
        r0, r1 = bnd[g], bnd[g + 1]
        assert P["n_local"] == r1 - r0
        cols = H.col[H.rowptr[r0]:H.rowptr[r1]]
        assert np.array_equal(P["ghosts"], np.unique(cols[(cols < r0) | (cols >= r1)]))
        for q in range(world):
            go, gc, so, sc = P["peers"][q]
            mine_from_q = P["ghosts"][go:go + gc]
            assert np.all((mine_from_q >= bnd[q]) & (mine_from_q < bnd[q + 1]))
            # what q sends to g == what g expects from q, in the same order
            qo, qc = plans[q]["peers"][g][2:]
            assert np.array_equal(plans[q]["send_rows"][qo:qo + qc] + bnd[q], mine_from_q)
        assert P["peers"][:, 1].sum() == len(P["ghosts"]) and P["peers"][:, 3].sum() == len(P["send_rows"])


def _worker(rank, world, port, case, out):
    import torch
    import torch.distributed as dist
    from paper_1105_5481_b200 import kpm
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    H = sparse_cases()[case]
    x = np.random.default_rng(5).normal(size=H.D)  # the same global vector on every rank
    P = kpm.kpm_csr_partition(H.D, H.rowptr, H.col, rank, world)
    r0 = block_bounds(H.D, world)[rank]
    nl = P["n_local"]
    xloc = x[r0:r0 + nl]
    ext = np.concatenate([xloc, np.zeros(len(P["ghosts"]))])
    reqs = []
    for q in range(world):  # the NCCL send/recv pattern of the library, over gloo
        go, gc, so, sc = P["peers"][q]
        if sc:
            reqs.append(dist.isend(torch.from_numpy(xloc[P["send_rows"][so:so + sc]].copy()), q))
        if gc:
            buf = torch.zeros(int(gc), dtype=torch.float64)
            reqs.append((dist.irecv(buf, q), buf, go))
    for rq in reqs:
        if isinstance(rq, tuple):
            rq[0].wait()
            ext[nl + rq[2]: nl + rq[2] + len(rq[1])] = rq[1].numpy()
        else:
            rq.wait()
    # local rows with extended-block column numbering
    gidx = {int(j): nl + k for k, j in enumerate(P["ghosts"])}
    y = np.zeros(nl)
    for i in range(nl):
        for e in range(H.rowptr[r0 + i], H.rowptr[r0 + i + 1]):
            j = int(H.col[e])
            jl = j - r0 if r0 <= j < r0 + nl else gidx[j]
            y[i] += H.val_re[e] * ext[jl]
    out[rank] = y.tolist()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("case", ["random", "lattice3d"])
def test_ghost_exchange_world2_gloo_reproduces_spmv(case):
    world = 2
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, _free_port(), case, out), nprocs=world, join=True)
    H = sparse_cases()[case]
    x = np.random.default_rng(5).normal(size=H.D)
    y = np.concatenate([np.asarray(out[g]) for g in range(world)])
    assert np.abs(y - H.dense().real @ x).max() < 1e-12
