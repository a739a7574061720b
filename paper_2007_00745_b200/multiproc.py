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


class RankRenderer:
    """Rank ``rank`` of ``world`` rendering one configuration into rank 0's map.

    ``args`` are the scalar arguments (xmin, xmax, ymin, ymax, W, H, iterMax, R);
    ``stream`` is the cudaStream_t (int) of this rank's device.
    """

    CTR_BYTES = 256

    def __init__(self, dist, rank: int, world: int, device: int, args, dtype: str, stream):
        self.dist, self.rank, self.world, self.device = dist, rank, world, device
        self.args, self.dtype, self.stream = tuple(args), dtype, stream
        W, H = int(args[4]), int(args[5])
        self.nbytes = W * H * 4
        self.owned = []
        self.mapped = []
        if rank == 0:
            self.img = M.mandel_dev_alloc(device, self.nbytes)
            self.ctr = M.mandel_dev_alloc(device, self.CTR_BYTES)
            self.owned = [self.img, self.ctr]
            handles = (M.mandel_ipc_handle(self.img), M.mandel_ipc_handle(self.ctr))
            share_bytes(dist, rank, handles)
        else:
            handles = share_bytes(dist, rank, None)
            self.img = M.mandel_ipc_open(device, handles[0])
            self.ctr = M.mandel_ipc_open(device, handles[1])
            self.mapped = [self.img, self.ctr]
        dist.barrier()

    def step(self, scheme: str, **kw) -> dict:
        """One render: reset the shared counter (FCFS), line up, render, line up."""
        if M.SCHEMES[scheme] in (M.MANDEL_FCFS, M.MANDEL_FCFS_MASTER) and self.rank == 0:
            M.mandel_dev_zero(self.ctr, self.CTR_BYTES, self.stream)
        self.dist.barrier()
        st = M.mandel_render_rank(*self.args, self.dtype, scheme, self.rank, self.world, self.img,
                                  self.ctr, self.stream, **kw)
        self.dist.barrier()
        return st

    def close(self):
        self.dist.barrier()
        for p in self.mapped:
            M.mandel_ipc_close(p)
        self.mapped = []
        self.dist.barrier()
        for p in self.owned:
            M.mandel_dev_free(p)
        self.owned = []
