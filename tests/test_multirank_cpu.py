"""The N > 1 host path on CPU: world_size 2 over gloo (127.0.0.1).

paper_1105_5481_b200.kpm.moments_distributed runs each rank's share of the vectors,
all-reduces the raw sums once and assembles mu.  Here the per-rank raw sums come from
the oracle (no GPU on this box), everything after that is the product path:
kpm_vector_range (partition), torch.distributed.all_reduce (gloo), kpm_assemble (C ABI,
host arithmetic).  The result must equal the oracle on all R vectors at once."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import kpm_inputs as ki
import oracle

N, R, SEED = 40, 7, 13
LAT = dict(ndim=2, L=(12, 9, 1), D=108, t=-1.0, onsite=ki.anderson_onsite(2, 108, 1.0), flux=0.0)


class OracleBackedHandle:
    """Stands in for kpm.Handle's raw-sum output on a CPU-only box."""

    def __init__(self, rank, world):
        from paper_1105_5481_b200 import kpm
        self.kpm = kpm
        self.D = LAT["D"]
        self.rank, self.world = rank, world
        H = oracle.lattice_csr(LAT)
        self.a, self.b = oracle.gershgorin(H)
        self.H = H

    def moments_ex(self, N_, R_, seed, flags=0):
        kpm = self.kpm
        assert flags & kpm.KPM_RAW_SUMS
        lo, cnt = kpm.kpm_vector_range(R_, self.rank, self.world)
        r = ki.rademacher(seed, cnt, self.D, r_offset=lo)
        _, pv = oracle.moments_doubling(self.H, self.a, self.b, r, N_, per_vector=True)
        # per-vector moments -> raw doubling sums: s_0 = D mu_0, s_1 = D mu_1,
        # s_2n = D (mu_2n + mu_0)/2, s_2n+1 = D (mu_2n+1 + mu_1)/2
        s = pv * self.D
        s[:, 2::2] = (s[:, 2::2] + s[:, [0]]) / 2
        s[:, 3::2] = (s[:, 3::2] + s[:, [1]]) / 2
        return s.sum(axis=0)

    def assemble(self, S, N_, R_, flags=0):
        return self.kpm.kpm_assemble_host(S, N_, self.D, R_, flags)


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1105_5481_b200 import kpm
    mu = kpm.moments_distributed(OracleBackedHandle(rank, world), N, R, SEED, device=torch.device("cpu"))
    out[rank] = mu.tolist()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
def test_vector_partition_allreduce_assemble(world):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    H = oracle.lattice_csr(LAT)
    a, b = oracle.gershgorin(H)
    ref = oracle.moments_doubling(H, a, b, ki.rademacher(SEED, R, LAT["D"]), N)
    for rank in range(world):
        assert np.abs(np.array(out[rank]) - ref).max() < 1e-13
    assert out[0] == out[world - 1]


def test_vector_range_tiles_all_vectors():
    from paper_1105_5481_b200 import kpm
    for R_, world in [(64, 8), (7, 3), (5, 5), (1000, 7)]:
        got = [kpm.kpm_vector_range(R_, r, world) for r in range(world)]
        assert got[0][0] == 0 and sum(c for _, c in got) == R_
        assert all(got[i][0] + got[i][1] == got[i + 1][0] for i in range(world - 1))


def test_assemble_host_transform():
    from paper_1105_5481_b200 import kpm
    S = np.array([10.0, 4.0, 7.0, 3.0, 9.0])
    mu = kpm.kpm_assemble_host(S, 5, 5, 2)
    c = 1 / 10
    assert np.allclose(mu, [1.0, 0.4, 2 * 0.7 - 1.0, 2 * 0.3 - 0.4, 2 * 0.9 - 1.0], rtol=0, atol=1e-15)
    assert np.allclose(kpm.kpm_assemble_host(S, 5, 5, 2, flags=kpm.KPM_DIRECT), S * c)


def _id_worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1105_5481_b200 import kpm
    out[rank] = kpm.nccl_id_for_group().hex()
    dist.destroy_process_group()


def test_row_partition_nccl_id_broadcast_over_gloo():
    """Plumbing of KPM_COMM_NCCL: rank 0's ncclUniqueId reaches every rank unchanged."""
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_id_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert out[0] == out[1] and len(out[0]) == 256


def test_slab_range_tiles_planes():
    from paper_1105_5481_b200 import kpm
    for Lm, world in [(512, 8), (10, 3), (7, 7), (128, 5)]:
        got = [kpm.kpm_slab_range(Lm, r, world) for r in range(world)]
        assert got[0][0] == 0 and sum(c for _, c in got) == Lm and min(c for _, c in got) >= 1
        assert all(got[i][0] + got[i][1] == got[i + 1][0] for i in range(world - 1))
