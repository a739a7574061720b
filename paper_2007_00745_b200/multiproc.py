"""One-process-per-GPU plumbing around mandel_render_rank (torch.distributed).

The paper's master-slave gather ("send the data back to the master
node") becomes: rank 0 owns the map and the FCFS chunk counter in its HBM; it
exports both as CUDA IPC handles, every other rank maps them, and each rank's
kernel stores its pixels straight into rank 0's map over NVLink
(mandel_render_rank).  torch.distributed carries only the handles, the
barriers and the timing reductions -- plumbing, not the data path.
"""
from __future__ import annotations

import numpy as np

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

    Step protocol.  Rank 0 owns ``slots`` FCFS counters (one per render, zeroed
    together); render n claims from counter n mod slots, so consecutive renders
    never share a counter and need no barrier between them: a rank that finishes
    render n early starts render n+1 at once (the map is rewritten with the same
    values).  When the slots run out, every rank lines up, rank 0 zeroes them all
    and every rank lines up again.  ``step(barrier=True)`` ends a render with a
    barrier -- needed when the caller reads the whole map right after it (e2e).
    """

    CTR_BYTES = 256

    def __init__(self, dist, rank: int, world: int, device: int, args, dtype: str, stream, lib=None,
                 slots: int = 512, images: int = 1):
        self.M = lib if lib is not None else M
        self.dist, self.rank, self.world, self.device = dist, rank, world, device
        self.args, self.dtype, self.stream = tuple(args), dtype, stream
        self.slots = slots
        W, H = int(args[4]), int(args[5])
        self.nbytes = W * H * 4
        self.owned = []
        self.mapped = []
        self.nstep = 0
        L = self.M
        # ``images`` maps on rank 0 (2: a render can proceed while the previous one is
        # drained to the host, bench.py's pipelined e2e)
        if rank == 0:
            self.imgs = [L.mandel_dev_alloc(device, self.nbytes) for _ in range(images)]
            ctr = L.mandel_dev_alloc(device, slots * self.CTR_BYTES)
            L.mandel_dev_zero(ctr, slots * self.CTR_BYTES, stream)
            self.owned = self.imgs + [ctr]
            handles = tuple(L.mandel_ipc_handle(p) for p in self.imgs) + (L.mandel_ipc_handle(ctr),)
            share_bytes(dist, rank, handles)
        else:
            handles = share_bytes(dist, rank, None)
            self.imgs = [L.mandel_ipc_open(device, h) for h in handles[:-1]]
            ctr = L.mandel_ipc_open(device, handles[-1])
            self.mapped = self.imgs + [ctr]
        self.img = self.imgs[0]
        self.ctr = ctr
        dist.barrier()

    def counter(self, n: int) -> int:
        return self.ctr + (n % self.slots) * self.CTR_BYTES

    def step(self, scheme: str, barrier: bool = False, sync: bool = True, image: int = 0, **kw):
        """One render into rank 0's map ``image`` (see the class notes for the protocol).
        sync=False only enqueues the render on the stream and returns None."""
        L = self.M
        if self.nstep and self.nstep % self.slots == 0:  # every counter used once: recycle
            L.mandel_sync(self.stream)  # earlier renders may still be claiming (sync=False)
            self.dist.barrier()
            if self.rank == 0:
                L.mandel_dev_zero(self.ctr, self.slots * self.CTR_BYTES, self.stream)
            self.dist.barrier()
        if not sync:
            kw["want_stats"] = False
        st = L.mandel_render_rank(*self.args, self.dtype, scheme, self.rank, self.world, self.imgs[image],
                                  self.counter(self.nstep), self.stream, **kw)
        self.nstep += 1
        if barrier:
            if not sync:  # the barrier orders host calls: the render must be finished first
                L.mandel_sync(self.stream)
            self.dist.barrier()
        return st

    def device_barrier(self):
        """Order every rank's next render after every rank's current one, ON THE DEVICE:
        a one-element all_reduce enqueued on the render stream (NCCL over NVLink, no host
        round trip), so a timed sequence of renders measures each render to the moment
        the last rank's stores have landed in rank 0's map -- the paper's compute time
        ends when the master holds the image (Eq. 21's T_N),
        FCFS tail included.  With gloo (the CPU plumbing of the tests) the stream is
        synchronised and the host barrier used instead."""
        if self.dist.get_backend() != "nccl":
            self.M.mandel_sync(self.stream)
            self.dist.barrier()
            return
        import torch
        dev = torch.device("cuda", self.device)
        if getattr(self, "_tok", None) is None:
            self._tok = torch.zeros(1, dtype=torch.int32, device=dev)
        with torch.cuda.stream(torch.cuda.ExternalStream(self.stream, device=dev)):
            self.dist.all_reduce(self._tok)

    def close(self):
        self.dist.barrier()
        for p in self.mapped:
            self.M.mandel_ipc_close(p)
        self.mapped = []
        self.dist.barrier()
        for p in self.owned:
            self.M.mandel_dev_free(p)
        self.owned = []


class GatherRenderer(RankRenderer):
    """The NCCL gather path (the cross-check of the fused peer stores).

    Each rank renders its rows into its own compact band (``band_out``: band row b =
    the rank's b-th row slot), then rank 0 receives every other rank's band and row
    list with point-to-point sends (torch.distributed P2P ops -- NCCL on a GPU job;
    with gloo, the CPU test plumbing, through host copies) and places each band in the
    image with K4 (``mandel_scatter_rows``), the paper's master "reconstructs the
    image".  FCFS claims still use rank 0's shared counter.
    """

    def __init__(self, dist, rank, world, device, args, dtype, stream, lib=None, slots=512,
                 chunk_rows=16):
        super().__init__(dist, rank, world, device, args, dtype, stream, lib=lib, slots=slots)
        import torch
        W, H = int(args[4]), int(args[5])
        self.W, self.H = W, H
        c = max(1, int(chunk_rows))
        self.cap = -(-H // c) * c  # band rows a rank may need (FCFS: every chunk)
        self.dev = torch.device("cuda", device)
        self.band = torch.empty((self.cap, W), dtype=torch.int32, device=self.dev)
        self.host = dist.get_backend() == "gloo"
        if rank == 0:
            self.recv = [torch.empty((self.cap, W), dtype=torch.int32, device=self.dev)
                         for _ in range(world)]

    def step(self, scheme: str, barrier: bool = False, sync: bool = True, **kw) -> dict:
        """One render + gather (always synchronous: the band's row list is read back)."""
        import torch
        L, dist = self.M, self.dist
        if self.nstep and self.nstep % self.slots == 0:
            L.mandel_sync(self.stream)
            dist.barrier()
            if self.rank == 0:
                L.mandel_dev_zero(self.ctr, self.slots * self.CTR_BYTES, self.stream)
            dist.barrier()
        st = L.mandel_render_rank(*self.args, self.dtype, scheme, self.rank, self.world,
                                  self.band.data_ptr(), self.counter(self.nstep), self.stream,
                                  band_out=True, **kw)
        self.nstep += 1
        rows = torch.from_numpy(L.mandel_band_rows().view(np.int32))
        cdev = torch.device("cpu") if self.host else self.dev
        n = torch.tensor([rows.numel()], dtype=torch.int64, device=cdev)
        counts = [torch.zeros(1, dtype=torch.int64, device=cdev) for _ in range(self.world)]
        dist.all_gather(counts, n)
        counts = [int(x.item()) for x in counts]
        W = self.W
        if self.rank == 0:
            bands = {0: (self.band, rows)}
            ops, recv_rows = [], {}
            for r in range(1, self.world):
                if counts[r] == 0:
                    continue
                rr = torch.empty(counts[r], dtype=torch.int32, device=cdev)
                dst = self.recv[r][:counts[r]] if not self.host else \
                    torch.empty((counts[r], W), dtype=torch.int32)
                ops += [dist.P2POp(dist.irecv, rr, r), dist.P2POp(dist.irecv, dst, r)]
                recv_rows[r] = (dst, rr)
            for w in (dist.batch_isend_irecv(ops) if ops else []):
                w.wait()
            for r, (dst, rr) in recv_rows.items():
                if self.host:
                    self.recv[r][:counts[r]].copy_(dst)
                    dst = self.recv[r][:counts[r]]
                bands[r] = (dst, rr)
            scatters = 0
            for r, (b, rw) in bands.items():
                if counts[r] == 0:
                    continue
                rd = rw.to(self.dev)
                L.mandel_scatter_rows(b.data_ptr(), rd.data_ptr(), counts[r], W, self.img, self.stream)
                scatters += 1
            torch.cuda.current_stream(self.dev).synchronize()
        elif counts[self.rank]:
            cnt = counts[self.rank]
            payload = self.band[:cnt] if not self.host else self.band[:cnt].cpu()
            rsend = rows if self.host else rows.to(self.dev)
            ops = [dist.P2POp(dist.isend, rsend, 0), dist.P2POp(dist.isend, payload, 0)]
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        if barrier:
            dist.barrier()
        st = dict(st)
        st["band_rows"] = counts[self.rank]
        if self.rank == 0:
            st["kernel_launches"] = st["kernel_launches"] + scatters  # K4 launches
        return st


class SharedHostImage:
    """The end-to-end destination of a one-process-per-GPU job: one host buffer shared by
    every rank (POSIX shared memory, page-locked in every process with cudaHostRegister),
    so that the hand-off of rank 0's map (the master's file write) uses
    every GPU's PCIe link: rank r copies rows [r*H/N, (r+1)*H/N) of rank 0's map -- over
    NVLink through its CUDA IPC mapping -- into the shared buffer.  ``ok`` is False when
    the segment cannot be created or registered; callers then copy from rank 0 alone.
    """

    def __init__(self, dist, rank: int, nbytes: int, cudart):
        from multiprocessing import shared_memory
        import ctypes
        self.dist, self.rank, self.nbytes, self.cudart = dist, rank, nbytes, cudart
        self.shm, self.ptr, self.ok = None, 0, False
        err = ""
        name = None
        if rank == 0:
            try:
                self.shm = shared_memory.SharedMemory(create=True, size=nbytes)
                name = self.shm.name
            except Exception as e:  # e.g. /dev/shm too small
                err = f"shm: {e}"[:120]
        name = share_bytes(dist, rank, name)
        if rank != 0 and name is not None:
            try:
                self.shm = shared_memory.SharedMemory(name=name)
            except Exception as e:
                err = f"shm attach: {e}"[:120]
        if self.shm is not None:
            buf = (ctypes.c_char * nbytes).from_buffer(self.shm.buf)
            self.ptr = ctypes.addressof(buf)
            del buf
            rc = cudart.cudaHostRegister(ctypes.c_void_p(self.ptr), ctypes.c_size_t(nbytes), ctypes.c_uint(1))
            if rc != 0:
                err = f"cudaHostRegister rc={rc}"
                self.ptr = 0
        ok = 1 if (self.ptr and not err) else 0
        import torch
        tdev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" \
            else torch.device("cpu")
        t = torch.tensor([ok], dtype=torch.int32, device=tdev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        self.ok = bool(t.item())
        self.error = err

    def rows(self, H: int, world: int):
        """The row range this rank drains."""
        r0 = H * self.rank // world
        return r0, H * (self.rank + 1) // world - r0

    def drain(self, img_ptr: int, W: int, H: int, world: int, stream: int, wait: bool = True) -> None:
        """Copy this rank's slice of rank 0's map (device pointer valid here) to the host
        on ``stream``; wait=False returns once the copy is enqueued."""
        import ctypes
        r0, n = self.rows(H, world)
        if n == 0:
            return
        off = r0 * W * 4
        rc = self.cudart.cudaMemcpyAsync(ctypes.c_void_p(self.ptr + off), ctypes.c_void_p(img_ptr + off),
                                         ctypes.c_size_t(n * W * 4), ctypes.c_int(2), ctypes.c_void_p(stream))
        if rc != 0:
            raise RuntimeError(f"cudaMemcpyAsync (shared host slice) failed: {rc}")
        if wait:
            self.cudart.cudaStreamSynchronize(ctypes.c_void_p(stream))

    def checksum(self) -> int:
        """Sum of the host image as uint32 counts (no buffer export outlives the call)."""
        a = np.ndarray((self.nbytes // 4,), dtype=np.uint32, buffer=self.shm.buf)
        total = int(a.sum(dtype=np.uint64))
        del a
        return total

    def close(self):
        import ctypes
        if self.ptr:
            self.cudart.cudaHostUnregister(ctypes.c_void_p(self.ptr))
            self.ptr = 0
        self.dist.barrier()
        if self.shm is not None:
            self.shm.close()
            if self.rank == 0:
                self.shm.unlink()
            self.shm = None
