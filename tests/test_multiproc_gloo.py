"""The one-process-per-GPU host logic under torch.distributed (gloo, world size 2,
CPU only): handle broadcast, max/sum timing reduction, and the library's static
row plans assembled across real processes (coverage = a permutation of rows)."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    from paper_2007_00745_b200 import mandel
    from paper_2007_00745_b200.multiproc import aggregate, share_bytes
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = {}
        # rank 0's (fake) IPC handles reach every rank byte for byte
        payload = (bytes(range(64)), bytes(reversed(range(64)))) if rank == 0 else None
        got = share_bytes(dist, rank, payload)
        out["handles_ok"] = got == (bytes(range(64)), bytes(reversed(range(64))))
        # whole-job timing: max over ranks of the time, sum of the iterations
        ms, iters = aggregate(dist, 10.0 + rank, 1000 * (rank + 1))
        out["agg"] = (ms, iters)
        # each rank plans its own rows with the C-ABI planner; gather and check coverage
        for scheme, H in (("block", 8000), ("cyclic", 8000), ("block", 1001), ("cyclic", 1001)):
            rows = mandel.mandel_plan_rows(scheme, H, world, rank).tolist()
            allrows = [None] * world
            dist.all_gather_object(allrows, rows)
            flat = sorted(r for part in allrows for r in part)
            out[f"{scheme}{H}"] = flat == list(range(H))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_two_rank_plumbing():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        assert res[r]["handles_ok"]
        assert res[r]["agg"] == (11.0, 3000)
        for k in ("block8000", "cyclic8000", "block1001", "cyclic1001"):
            assert res[r][k], k
