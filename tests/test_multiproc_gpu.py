"""The one-process-per-GPU path bench.py runs under torchrun, on the one GPU a test box
has: 2-3 processes (gloo for the plumbing) each drive mandel_render_rank on cuda:0,
rank 0's map and FCFS counters exported with CUDA IPC and mapped by the others, every
rank's kernel storing straight into rank 0's map.  The ranks never wait on one another
(FCFS claims are non-blocking atomics), so sharing one device is safe; what this checks
is the plumbing (IPC handles, counter alternation, system-scope claims, fused stores),
compared bit for bit with the oracle."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import workloads as wl

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, cfg, schemes, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import bench
    from paper_2007_00745_b200 import mandel as M
    from paper_2007_00745_b200.multiproc import RankRenderer, aggregate
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        stream = torch.cuda.current_stream(0).cuda_stream
        rr = RankRenderer(dist, rank, world, 0, cfg.args(), cfg.dtype, stream, slots=4)
        res = {}
        for scheme in schemes:
            for rep in range(3):  # several renders: counter slots are used in turn and recycled
                if rank == 0:  # a zeroed map: every pixel must be (re)written by some rank
                    M.mandel_dev_zero(rr.img, cfg.W * cfg.H * 4, stream)
                dist.barrier()
                st = rr.step(scheme, barrier=True)
                _, iters = aggregate(dist, st["kernel_ms_max"], st["sum_iters"])
                if rank == 0:
                    host = torch.empty((cfg.H, cfg.W), dtype=torch.int32, pin_memory=True)
                    bench._d2h(host, rr.img, cfg.W * cfg.H * 4, stream)
                    res[(scheme, rep)] = (host.numpy().view(np.uint32).copy(), iters)
                dist.barrier()
        rr.close()
        q.put((rank, res))
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
def test_rank_processes_share_one_map(oracle, world, dtype):
    cfg = wl.C1.with_(dtype=dtype, W=517, H=389, iter_max=1500)
    want = oracle.render(cfg)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    schemes = ("fcfs", "cyclic", "block")
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, schemes, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0, res
    got = res[0]
    assert isinstance(got, dict), got
    for (scheme, rep), (img, iters) in got.items():
        bad = int((img != want).sum())
        assert bad == 0, f"{scheme} step {rep}: {bad} pixels differ from the oracle"
        assert iters == int(want.sum(dtype=np.uint64)), (scheme, rep)
