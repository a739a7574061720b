"""One-process-per-GPU plumbing around mandel_render_rank (torch.distributed).

The paper's master-slave gather ("send the data back to the master
node") becomes: rank 0 owns the map and the FCFS chunk counter in its HBM; it
exports both as CUDA IPC handles, every other rank maps them, and each rank's
kernel stores its pixels straight into rank 0's map over NVLink
(mandel_render_rank).  torch.distributed carries only the handles, the
barriers and the timing reductions -- plumbing, not the data path.
"""
from __future__ import annotations

from . import mandel as M


def share_bytes(dist, rank: int, payload, src: int = 0):
    """Broadcast a picklable payload (e.g. IPC handle bytes) from ``src``."""
    obj = [payload if rank == src else None]
    dist.broadcast_object_list(obj, src=src)
    return obj[0]


def aggregate(dist, rank_ms: float, rank_iters: int, device=None):
    """Whole-job numbers: max over ranks of a time, sum over ranks of a count."""
    if dist is None:
        return rank_ms, rank_iters
    import torch
    t = torch.tensor([rank_ms], dtype=torch.float64, device=device)
    n = torch.tensor([rank_iters], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(n, op=dist.ReduceOp.SUM)
    return float(t.item()), int(n.item())


def sum_over_ranks(dist, values, device=None):
    """Element-wise sum over ranks of a list of integers (e.g. per-step iteration counts)."""
    if dist is None:
        return [int(v) for v in values]
    import torch
    t = torch.tensor([int(v) for v in values], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [int(v) for v in t.tolist()]


class RankRenderer:
    """Rank ``rank`` of ``world`` rendering one configuration into rank 0's map.

    ``args`` are the scalar arguments (xmin, xmax, ymin, ymax, W, H, iterMax, R);
    ``stream`` is the cudaStream_t (int) of this rank's device.  ``lib`` is the
    binding module (tests pass a recording stand-in to check the step protocol).

    Step protocol (one barrier per render): the FCFS counter alternates between
    two slots by step parity.  During step s rank 0 zeroes the slot step s+1 will
    use (stream-ordered and synchronised before its render returns); the barrier
    that ends step s then orders that zero before every rank's first claim of
    step s+1, and no rank still claims from that slot (it was step s-1's, which
    every rank finished before the previous barrier).
    """

    CTR_BYTES = 256

    def __init__(self, dist, rank: int, world: int, device: int, args, dtype: str, stream, lib=None):
        self.M = lib if lib is not None else M
        self.dist, self.rank, self.world, self.device = dist, rank, world, device
        self.args, self.dtype, self.stream = tuple(args), dtype, stream
        W, H = int(args[4]), int(args[5])
        self.nbytes = W * H * 4
        self.owned = []
        self.mapped = []
        self.nstep = 0
        L = self.M
        if rank == 0:
            self.img = L.mandel_dev_alloc(device, self.nbytes)
            ctr = L.mandel_dev_alloc(device, 2 * self.CTR_BYTES)
            L.mandel_dev_zero(ctr, 2 * self.CTR_BYTES, stream)
            self.owned = [self.img, ctr]
            handles = (L.mandel_ipc_handle(self.img), L.mandel_ipc_handle(ctr))
            share_bytes(dist, rank, handles)
        else:
            handles = share_bytes(dist, rank, None)
            self.img = L.mandel_ipc_open(device, handles[0])
            ctr = L.mandel_ipc_open(device, handles[1])
            self.mapped = [self.img, ctr]
        self.ctrs = (ctr, ctr + self.CTR_BYTES)
        dist.barrier()

    def step(self, scheme: str, **kw) -> dict:
        """One render: rank 0 readies the next step's counter, every rank renders, line up."""
        L = self.M
        cur, nxt = self.ctrs[self.nstep % 2], self.ctrs[(self.nstep + 1) % 2]
        if self.rank == 0:
            L.mandel_dev_zero(nxt, self.CTR_BYTES, self.stream)
        st = L.mandel_render_rank(*self.args, self.dtype, scheme, self.rank, self.world, self.img,
                                  cur, self.stream, **kw)
        self.dist.barrier()
        self.nstep += 1
        return st

    def close(self):
        self.dist.barrier()
        for p in self.mapped:
            self.M.mandel_ipc_close(p)
        self.mapped = []
        self.dist.barrier()
        for p in self.owned:
            self.M.mandel_dev_free(p)
        self.owned = []
