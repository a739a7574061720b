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
        out["protocol"] = _step_protocol(dist, rank, world)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


class _RecordingLib:
    """Stands in for the binding in RankRenderer: records the calls in order."""
    MANDEL_FCFS = 2

    def __init__(self, log):
        self.log, self.next = log, 0x10000

    def mandel_dev_alloc(self, device, nbytes):
        self.next += 0x100000
        self.log.append(("alloc", self.next, nbytes))
        return self.next

    def mandel_dev_zero(self, ptr, nbytes, stream):
        self.log.append(("zero", ptr, nbytes))

    def mandel_ipc_handle(self, ptr):
        return ptr.to_bytes(64, "little")

    def mandel_ipc_open(self, device, h):
        return int.from_bytes(h, "little")

    def mandel_ipc_close(self, ptr):
        self.log.append(("close", ptr))

    def mandel_dev_free(self, ptr):
        self.log.append(("free", ptr))

    def mandel_sync(self, stream):
        self.log.append(("sync",))

    def mandel_render_rank(self, *a, **kw):
        self.log.append(("render", a[13], a[12]))  # (counter pointer, image pointer)
        return {}


def _step_protocol(dist, rank, world):
    """RankRenderer's step protocol: one zeroed counter slot per render, no barrier between
    renders, all slots recycled (barrier, zero, barrier) when used up; barrier=True ends a
    render with a barrier."""
    from paper_2007_00745_b200.multiproc import RankRenderer
    log = []
    real_barrier = dist.barrier

    class D:
        def __getattr__(self, k):
            return getattr(dist, k)

        def barrier(self):
            log.append(("barrier",))
            real_barrier()

    rr = RankRenderer(D(), rank, world, 0, (-2.5, 1.5, -2.0, 2.0, 64, 48, 100, 2.0), "fp64", 0,
                      lib=_RecordingLib(log), slots=3)
    B = rr.CTR_BYTES
    ok = True
    if rank == 0:  # all three slots zeroed once at set-up
        ok = ok and ("zero", rr.ctr, 3 * B) in log
    n0 = len(log)
    for _ in range(7):
        rr.step("fcfs")
    rr.step("fcfs", barrier=True)
    steps = log[n0:]
    want = []
    for n in range(8):
        if n and n % 3 == 0:
            want += [("sync",), ("barrier",)] + ([("zero", rr.ctr, 3 * B)] if rank == 0 else []) + \
                [("barrier",)]
        want.append(("render", rr.ctr + (n % 3) * B, rr.img))
    want.append(("barrier",))
    ok = ok and steps == want
    # device_barrier: on the CPU plumbing (gloo) it synchronises the stream, then lines up
    n1 = len(log)
    rr.step("block", sync=False)
    rr.device_barrier()
    ok = ok and log[n1:] == [("render", rr.ctr + (8 % 3) * B, rr.img), ("sync",), ("barrier",)]
    rr.close()
    return ok


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
        assert res[r]["protocol"]
