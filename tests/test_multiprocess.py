"""The N>1 plumbing on CPU: two gloo ranks exercise bench.py's rank reduction (max of the device
time, tokens summed for replicas or taken from rank 0 under expert parallelism) and the NCCL-id
broadcast path (with a stand-in id), as torchrun would launch them."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    ms, toks = bench.reduce_over_ranks(10.0 + rank, 100 + rank, sum_tokens=True)
    ms2, toks2 = bench.reduce_over_ranks(5.0 * (rank + 1), 7 + rank, sum_tokens=False)
    obj = [b"id-bytes" if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    assert bench.dist_env()[:2] == (rank, world)
    q.put((rank, ms, toks, ms2, toks2, obj[0]))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_rank_reduction():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    [p.start() for p in procs]
    [p.join(timeout=120) for p in procs]
    assert all(p.exitcode == 0 for p in procs)
    got = sorted(q.get() for _ in range(2))
    for rank, ms, toks, ms2, toks2, oid in got:
        assert ms == 11.0 and toks == 201        # replicas: max time, summed tokens
        assert ms2 == 10.0 and toks2 == 7        # expert parallel: max time, rank-0 tokens
        assert oid == b"id-bytes"


def _host_worker(rank, world, port, q):
    """The C ABI's host transport callback (what the engine calls for every EP collective) over gloo."""
    import ctypes as C
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    from paper_2604_10152_b200.engine import HostTransport, gloo_allgather
    t = HostTransport(gloo_allgather())
    ok = []
    for n in (1, 40, 4099):
        send = (C.c_ubyte * n)(*[(rank * 31 + i) % 251 for i in range(n)])
        recv = (C.c_ubyte * (n * world))()
        rc = t.cfunc(None, C.addressof(send), C.addressof(recv), n)
        want = [(r * 31 + i) % 251 for r in range(world) for i in range(n)]
        ok.append(rc == 0 and list(recv) == want)
    q.put((rank, all(ok)))
    dist.barrier()
    dist.destroy_process_group()


def test_host_transport_allgather_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_host_worker, args=(r, 2, port, q)) for r in range(2)]
    [p.start() for p in procs]
    [p.join(timeout=120) for p in procs]
    assert all(p.exitcode == 0 for p in procs)
    assert sorted(q.get() for _ in range(2)) == [(0, True), (1, True)]
