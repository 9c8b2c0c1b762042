"""Worker processes for the multi-rank tests (spawned by tests/test_dist_*.py)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def _init(rank, world, port, backend="gloo"):
    import torch.distributed as dist

    dist.init_process_group(backend, init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    return dist


def cpu_comm_worker(rank, world, port, out_dir):
    """Exercise TorchComm's callbacks on host buffers (no GPU): allgather and the
    two-phase neighbour exchange the CUDA library performs (solver.cu neighbor_exchange)."""
    dist = _init(rank, world, port)
    from paper_2504_11167_b200.dist import TorchComm

    comm = TorchComm(device_buffers=False)
    res = {}
    # allgather: recv[q*count:(q+1)*count] = send of rank q
    count = 5
    send = np.arange(count, dtype=np.float64) + 100 * rank
    recv = np.zeros(count * world)
    assert comm._allgather(None, send.ctypes.data, recv.ctypes.data, count) == 0
    res["allgather"] = recv.copy()
    # phase A: to next / from prev; phase B: to prev / from next
    nxt = rank + 1 if rank + 1 < world else -1
    prv = rank - 1 if rank > 0 else -1
    to_next = np.full(3, 10.0 * rank + 1)
    to_prev = np.full(3, 10.0 * rank + 2)
    from_prev = np.full(3, -1.0)
    from_next = np.full(3, -1.0)
    assert comm._sendrecv(None, to_next.ctypes.data, 3 if nxt >= 0 else 0, nxt,
                          from_prev.ctypes.data, 3 if prv >= 0 else 0, prv) == 0
    assert comm._sendrecv(None, to_prev.ctypes.data, 3 if prv >= 0 else 0, prv,
                          from_next.ctypes.data, 3 if nxt >= 0 else 0, nxt) == 0
    res["from_prev"] = from_prev.copy()
    res["from_next"] = from_next.copy()
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **res)
    dist.barrier()
    dist.destroy_process_group()


def gpu_solve_worker(rank, world, port, out_dir, name, scale, method, P, variant="T",
                     backend="gloo"):
    """One rank of a sharded factorize + solve on cuda:0 (ranks share the GPU; all
    cross-rank dependencies are host-synchronous gloo calls).  backend="nccl" (one rank:
    NCCL refuses two ranks on one device) runs the adapter's device-buffer path."""
    dist = _init(rank, world, port, "gloo" if backend == "libnccl" else backend)
    import torch

    from paper_2504_11167_b200 import api, configs
    from paper_2504_11167_b200.dist import DistFactorization, LibNcclComm, TorchComm, gather_rows

    torch.cuda.set_device(0)
    cfg = configs.make_config(name, scale, P)
    ctx = api.Context(0)
    # libnccl: the in-library NCCL data plane (torch.distributed/gloo only shares the id)
    comm = LibNcclComm(ctx) if backend == "libnccl" else TorchComm(device_buffers=True)
    A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
    scfg = api.SolverConfig(variant=variant, p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed)
    F = DistFactorization(ctx, A, scfg, comm)
    f = np.asfortranarray(configs.vector("uniform", 77, cfg.matrix.n))
    y = F.apply_precond_T(f)
    it = api.IterConfig(tol=cfg.tol, method=method, restart=cfg.m or 30, max_iters=500)
    x, rep, _ = api.solve(A, np.asfortranarray(cfg.rhs), it=it, F=F)
    xg = gather_rows(x, F.row_lo, F.row_hi, cfg.matrix.n, comm)
    yg = gather_rows(y, F.row_lo, F.row_hi, cfg.matrix.n, comm)
    adapter = np.zeros(0)
    if backend == "nccl":
        # the library makes no exchanges on one rank: drive the device-buffer callbacks
        # directly (all-gather, and a send / receive to this rank itself)
        s = torch.arange(6, dtype=torch.float64, device="cuda") + 1.0
        r = torch.zeros(6 * world, dtype=torch.float64, device="cuda")
        assert comm._allgather(None, s.data_ptr(), r.data_ptr(), 6) == 0
        r2 = torch.zeros(6, dtype=torch.float64, device="cuda")
        assert comm._sendrecv(None, s.data_ptr(), 6, rank, r2.data_ptr(), 6, rank) == 0
        adapter = np.concatenate([r.cpu().numpy(), r2.cpu().numpy()])
    if backend == "libnccl":
        # one rank: drive the library's stream-ordered NCCL callbacks directly (all-gather,
        # a send / receive to this rank itself, and the grouped two-direction exchange)
        s = torch.arange(6, dtype=torch.float64, device="cuda") + 1.0
        r = torch.zeros(6 * world, dtype=torch.float64, device="cuda")
        r2 = torch.zeros(6, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        c = comm.c
        assert c.stream_ordered == 1
        assert c.allgather(c.user, s.data_ptr(), r.data_ptr(), 6) == 0
        assert c.sendrecv(c.user, s.data_ptr(), 6, rank, r2.data_ptr(), 6, rank) == 0
        ctx.synchronize()
        adapter = np.concatenate([r.cpu().numpy(), r2.cpu().numpy()])
    if rank == 0:
        np.savez(os.path.join(out_dir, "dist.npz"), x=xg, y=yg, iterations=rep.iterations,
                 adapter=adapter,
                 residual=rep.residual_final, history=np.array(rep.residual_history),
                 ledger=np.array([rep.comm["precond-apply"][1], rep.comm["recovery"][1]]),
                 calls=np.array([comm.calls["allgather"], comm.calls["sendrecv"]])
                 if hasattr(comm, "calls") else np.array([0, 0]),
                 round_trips=np.array([rep.round_trips["comm_calls"],
                                       rep.round_trips["comm_host_syncs"]]))
    dist.barrier()
    del F
    if backend == "libnccl":
        comm.close()
    dist.destroy_process_group()
