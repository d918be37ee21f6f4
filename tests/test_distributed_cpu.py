"""The N > 1 path on CPU: two gloo ranks (127.0.0.1) exercise the host-side plumbing of
the distributed evaluation -- the NCCL unique id made by the C ABI on rank 0 reaches
every rank bit-identically through torch.distributed, and bench.py's max-over-ranks
timing reduction. The device-side distributed schedule itself is covered on one GPU by
virtual ranks (tests/test_gpu_parity.py::test_virtual_ranks_*) and by the host-side
enumeration/ownership check (tests/test_host_logic.py)."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    import paper_1708_02835_b200 as ex

    nid = ex.exchange_nccl_id(rank, world)
    gathered = [None] * world
    dist.all_gather_object(gathered, nid)
    ms = bench.reduce_max(10.0 + rank, dist)
    env = bench.dist_env()
    dist.destroy_process_group()
    q.put((rank, len(nid), all(g == nid for g in gathered), ms, env))


def test_two_rank_gloo_plumbing():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, nbytes, same, ms, env in out:
        assert nbytes == 128 and same
        assert ms == 11.0  # max over ranks of 10 + rank
        assert env == (rank, world, rank)


def _grid_worker(rank, world, port, q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1708_02835_b200 as ex

    res = []
    for n, nb, P in [(10_000, 256, 2), (10_000, 256, 1), (3_001, 128, 4), (300_000, 512, 2)]:
        if world % P:
            continue
        Q = world // P
        p, qq = rank // Q, rank % Q
        # this process's share under the ownership rule tile (I, J) -> rank (I mod P, J mod Q),
        # written out independently of the library
        T = -(-n // nb)
        mine = 0
        for J in range(qq, T, Q):
            tiles = sum(1 for I in range(J, T) if I % P == p)
            mine += 8 * nb * (tiles * nb + (128 if T % P == p else 0))
        got = ex.rank_workspace_bytes(n, nb, world, P, rank)
        t = torch.tensor([got], dtype=torch.float64)
        dist.all_reduce(t)
        res.append((n, nb, P, got == mine + 2048, int(t.item()) == ex.workspace_bytes(n, nb) + 2048 * (world - 1)))
    dist.destroy_process_group()
    q.put((rank, res))


@pytest.mark.parametrize("world", [2, 4])
def test_grid_ownership_across_processes(world):
    """world gloo processes, one per rank of a P x Q grid: each rank's workspace (the C ABI's
    2-D block-cyclic layout) equals the tiles the ownership rule assigns to it, and the ranks'
    shares all-reduce to the single-GPU workspace -- every tile stored exactly once."""
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_grid_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, res in out:
        assert res
        for n, nb, P, own_ok, sum_ok in res:
            assert own_ok, (rank, n, nb, P)
            assert sum_ok, (rank, n, nb, P)
