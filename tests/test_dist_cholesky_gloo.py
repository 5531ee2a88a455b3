"""World-size 2 / 3 gloo run of the distributed factorisation's schedule (SHARD_CYCLIC, DESIGN.md
7.1) on CPU, in real processes: the same steps as dist_potrf / dist_potrs in csrc/ipm.cu with
torch.distributed.broadcast in place of ncclBroadcast and plain torch CPU tile ops in place of
cuSOLVER / cuBLAS.  Each rank holds only the pair tiles polya_plan(SHARD_CYCLIC) gives it
(npairs_local of them: block columns h = r mod N of the lower factor); the factor + solve must
reproduce a dense solve of the whole matrix.  (The GPU code itself runs the same steps in
tests/test_gpu_dist.py through the in-process loopback.)"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _spd(T, N, seed):
    rng = np.random.default_rng(seed)
    R = rng.normal(size=(T * N, T * N + 3))
    return R @ R.T / (T * N) + np.eye(T * N), rng.normal(size=T * N)


def _worker(rank, world, port, q, T, N, seed):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    G, b = _spd(T, N, seed)
    owner = lambda k: k % world
    # the pair tiles this rank holds: (h, h') with h = rank mod world; tile (k, i) = lower block B_ik
    tiles = {(h, h2): torch.tensor(G[h2 * N:(h2 + 1) * N, h * N:(h + 1) * N].copy())
             for h in range(T) if owner(h) == rank for h2 in range(h, T)}
    # dist_potrf
    for k in range(T):
        o = owner(k)
        info = torch.zeros(1, dtype=torch.int32)
        if rank == o:
            try:
                tiles[(k, k)] = torch.linalg.cholesky(tiles[(k, k)])
            except RuntimeError:
                info[0] = 1
        dist.broadcast(info, o)
        assert info[0] == 0
        if k + 1 == T:
            break
        # L_kk and the raw panel from the owner; the panel solves B_ik <- B_ik L_kk^{-T} split over the
        # ranks (tile q = i-k-1 on rank q mod N); the solved tiles broadcast from their solvers
        Lkk = tiles[(k, k)].contiguous().clone() if rank == o else torch.zeros(N, N, dtype=torch.float64)
        dist.broadcast(Lkk, o)
        panel = torch.stack([tiles[(k, i)] for i in range(k + 1, T)]) if rank == o else torch.zeros(T - k - 1, N, N,
                                                                                                  dtype=torch.float64)
        dist.broadcast(panel, o)
        for t in range(rank, T - k - 1, world):
            panel[t] = torch.linalg.solve_triangular(Lkk, panel[t].T, upper=False).T
        for t in range(T - k - 1):
            tt = panel[t].clone()
            dist.broadcast(tt, t % world)
            panel[t] = tt
        if rank == o:
            for i in range(k + 1, T):
                tiles[(k, i)] = panel[i - k - 1].clone()
        for j in range(k + 1, T):   # dist_update: this rank's block columns j > k
            if owner(j) != rank:
                continue
            Bjk = panel[j - k - 1]
            tiles[(j, j)] = tiles[(j, j)] - Bjk @ Bjk.T
            for i in range(j + 1, T):
                tiles[(j, i)] = tiles[(j, i)] - panel[i - k - 1] @ Bjk.T
    # dist_potrs
    x = torch.tensor(b.copy())
    for k in range(T):
        o = owner(k)
        if rank == o:
            x[k * N:(k + 1) * N] = torch.linalg.solve_triangular(tiles[(k, k)], x[k * N:(k + 1) * N, None], upper=False)[:, 0]
            for i in range(k + 1, T):
                x[i * N:(i + 1) * N] -= tiles[(k, i)] @ x[k * N:(k + 1) * N]
        seg = x[k * N:].clone()
        dist.broadcast(seg, o)
        x[k * N:] = seg
    for k in range(T - 1, -1, -1):
        o = owner(k)
        if rank == o:
            for i in range(k + 1, T):
                x[k * N:(k + 1) * N] -= tiles[(k, i)].T @ x[i * N:(i + 1) * N]
            x[k * N:(k + 1) * N] = torch.linalg.solve_triangular(tiles[(k, k)].T, x[k * N:(k + 1) * N, None], upper=True)[:, 0]
        seg = x[k * N:(k + 1) * N].clone()
        dist.broadcast(seg, o)
        x[k * N:(k + 1) * N] = seg
    out = [torch.zeros_like(x) for _ in range(world)]
    dist.all_gather(out, x)
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        q.put((len(tiles), [o.numpy() for o in out]))


@pytest.mark.parametrize("world,T", [(2, 5), (3, 6)])
def test_distributed_cholesky_schedule_gloo(world, T):
    import paper_1411_3769_b200 as pb
    N, seed = 7, world
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, T, N, seed)) for r in range(world)]
    for p in procs:
        p.start()
    ntiles0, xs = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    G, b = _spd(T, N, seed)
    ref = np.linalg.solve(G, b)
    for x in xs:   # every rank ends with the whole solution
        assert np.linalg.norm(x - ref) <= 1e-10 * np.linalg.norm(ref)
    # rank 0 held exactly the tiles polya_plan(SHARD_CYCLIC) assigns it: the pair rows h = 0 mod N
    # of an L0 = T problem (n = 1, l = T, dp = 1 gives L0 = T and Ntil = 1)
    assert pb.plan(1, T, 1, 1, 1, rank=0, nranks=world, shard=pb.SHARD_CYCLIC)["npairs_local"] == ntiles0
