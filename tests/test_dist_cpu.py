"""Multi-rank host logic on CPU (gloo, world_size 2 and 3): the shard plan, the
exchange callbacks of paper_2504_11167_b200.dist.TorchComm, and the partition-ordered
reduction that makes every GPU count produce bit-identical dot products."""
import os
import random
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

from tests import dist_worker


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("n,P,G", [(1000, 8, 1), (1000, 8, 2), (1003, 8, 3), (65536, 4, 4),
                                   (884736, 64, 8), (262144, 8, 8)])
def test_shard_plan(n, P, G):
    from paper_2504_11167_b200.dist import shard_plan

    prev_p, prev_r = 0, 0
    counts = []
    for rank in range(G):
        plo, phi, rlo, rhi = shard_plan(n, P, G, rank)
        assert plo == prev_p and rlo == prev_r  # contiguous, in rank order
        assert phi > plo and rhi > rlo
        counts.append(phi - plo)
        prev_p, prev_r = phi, rhi
    assert prev_p == P and prev_r == n
    assert max(counts) - min(counts) <= 1


@pytest.mark.parametrize("world", [2, 3])
def test_torchcomm_exchange_semantics(world):
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(dist_worker.cpu_comm_worker, args=(world, _port(), d), nprocs=world, join=True)
        for rank in range(world):
            z = np.load(os.path.join(d, f"rank{rank}.npz"))
            expect = np.concatenate([np.arange(5.0) + 100 * q for q in range(world)])
            assert np.array_equal(z["allgather"], expect)
            if rank > 0:  # phase A delivers the left neighbour's to_next
                assert np.all(z["from_prev"] == 10.0 * (rank - 1) + 1)
            else:
                assert np.all(z["from_prev"] == -1.0)
            if rank + 1 < world:  # phase B delivers the right neighbour's to_prev
                assert np.all(z["from_next"] == 10.0 * (rank + 1) + 2)
            else:
                assert np.all(z["from_next"] == -1.0)


def test_partition_ordered_reduction_is_gpu_count_invariant():
    """Mirror of krylov.cu: chunk partials -> per-partition sums (chunk order) -> all-gather
    -> sum over global partitions in order.  Any sharding gives the same bits."""
    from paper_2504_11167_b200.dist import shard_plan

    rng = random.Random(0)
    P = 8
    chunks = [[rng.uniform(-1, 1) * 10 ** rng.randint(-8, 8) for _ in range(rng.randint(1, 6))]
              for _ in range(P)]

    def total(G):
        blocks = []
        for rank in range(G):
            plo, phi, _, _ = shard_plan(10_000, P, G, rank)
            per = []
            for p in range(plo, phi):
                s = 0.0
                for c in chunks[p]:
                    s += c
                per.append(s)
            blocks.append(per)
        out = 0.0
        for per in blocks:  # gathered in rank order = global partition order
            for s in per:
                out += s
        return out

    ref = total(1)
    for G in (2, 3, 4, 8):
        assert total(G) == ref  # bitwise
