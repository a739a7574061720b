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


def _worker(rank, world, port, cfg, schemes, q, gather="fused"):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import bench
    from paper_2007_00745_b200 import mandel as M
    from paper_2007_00745_b200.multiproc import GatherRenderer, RankRenderer, aggregate
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        stream = torch.cuda.current_stream(0).cuda_stream
        cls = GatherRenderer if gather == "nccl" else RankRenderer
        rr = cls(dist, rank, world, 0, cfg.args(), cfg.dtype, stream, slots=4)
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


@pytest.mark.parametrize("gather", ["fused", "nccl"])
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
def test_rank_processes_share_one_map(oracle, world, dtype, gather):
    cfg = wl.C1.with_(dtype=dtype, W=517, H=389, iter_max=1500)
    want = oracle.render(cfg)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    schemes = ("fcfs", "cyclic", "block")
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, schemes, q, gather))
             for r in range(world)]
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


BAND_CASES = [(s, k) for s in ("block", "cyclic", "fcfs", "fcfs_master") for k in ("refill", "lazy2")] + \
    [("block", "static"), ("cyclic", "static")]


@pytest.mark.parametrize("scheme,kernel", BAND_CASES, ids=[f"{s}-{k}" for s, k in BAND_CASES])
@pytest.mark.parametrize("nranks", [2, 3, 5])
def test_band_mode_and_scatter(mandel, oracle, scheme, kernel, nranks):
    """The NCCL path's device pieces in one process: each rank renders its compact band
    (band_out), mandel_band_rows lists the band's image rows, K4 places it.  The band is
    sized exactly as the header documents (static: the plan's rows; FCFS: every chunk),
    so a kernel that stores at image rows instead of band rows writes out of bounds or
    leaves band rows unwritten (the static kernel did)."""
    import torch
    cfg = wl.C1.with_(W=301, H=203, iter_max=800)
    want = oracle.render(cfg)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev).cuda_stream
    image = torch.zeros((cfg.H, cfg.W), dtype=torch.int32, device=dev)
    ctr = torch.zeros(64, dtype=torch.int32, device=dev)
    chunk = 1 if scheme == "fcfs_master" else 16
    seen = []
    for r in range(nranks):
        if scheme in ("block", "cyclic"):
            cap = len(mandel.mandel_plan_rows(scheme, cfg.H, nranks, r))
        else:
            cap = -(-cfg.H // chunk) * chunk
        # one guard row past the documented capacity: it must stay untouched
        buf = torch.full((cap + 1, cfg.W), -7, dtype=torch.int32, device=dev)
        band = buf[:cap]
        st = mandel.mandel_render_rank(*cfg.args(), "fp64", scheme, r, nranks, band, ctr, stream,
                                       band_out=True, kernel=kernel)
        assert bool((buf[cap] == -7).all()), "band_out wrote past the band's capacity"
        rows = mandel.mandel_band_rows()
        if scheme in ("block", "cyclic"):
            assert rows.tolist() == mandel.mandel_plan_rows(scheme, cfg.H, nranks, r).tolist()
        valid = rows[rows != 0xFFFFFFFF]
        seen += valid.tolist()
        assert st["rank_rows"][0] == len(valid)
        # written band rows hold the oracle's rows; unused slots were never written
        got = band[: len(rows)].cpu().numpy().view(np.uint32)
        for b, row in enumerate(rows.tolist()):
            if row != 0xFFFFFFFF:
                assert np.array_equal(got[b], want[row]), (scheme, r, b, row)
            else:
                assert (got[b] == np.uint32(0xFFFFFFF9)).all()
        if len(rows):
            rd = torch.from_numpy(rows.view(np.int32)).to(dev)
            mandel.mandel_scatter_rows(band, rd, len(rows), cfg.W, image, stream)
    torch.cuda.synchronize()
    assert sorted(seen) == list(range(cfg.H))
    got = image.cpu().numpy().view(np.uint32)
    assert np.array_equal(got, want)


def _shared_worker(rank, world, port, cfg, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import bench
    from paper_2007_00745_b200.multiproc import RankRenderer, SharedHostImage
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        stream = torch.cuda.current_stream(0).cuda_stream
        rr = RankRenderer(dist, rank, world, 0, cfg.args(), cfg.dtype, stream, slots=4)
        sh = SharedHostImage(dist, rank, cfg.W * cfg.H * 4, bench._cudart())
        res = {"ok": sh.ok, "err": sh.error}
        if sh.ok:
            for scheme in ("fcfs", "cyclic"):
                rr.step(scheme, barrier=True)
                sh.drain(rr.img, cfg.W, cfg.H, world, stream)
                dist.barrier()
                if rank == 0:
                    a = np.ndarray((cfg.H, cfg.W), dtype=np.uint32, buffer=sh.shm.buf).copy()
                    res[scheme] = a
                dist.barrier()
        sh.close()
        rr.close()
        q.put((rank, res))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_shared_host_image_drain(oracle, world):
    """N > 1 end to end: every rank copies its slice of rank 0's map (through its CUDA IPC
    mapping) into one shared page-locked host image; the image equals the oracle's map."""
    cfg = wl.C1.with_(W=389, H=211, iter_max=900)
    want = oracle.render(cfg)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shared_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0, res
    got = res[0]
    assert isinstance(got, dict), got
    assert got["ok"], got["err"]
    for scheme in ("fcfs", "cyclic"):
        assert np.array_equal(got[scheme], want), scheme


def _probe_worker(rank, world, port, cfg, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import bench
    from paper_2007_00745_b200 import mandel as M
    from paper_2007_00745_b200.multiproc import RankRenderer
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        stream = torch.cuda.current_stream(0).cuda_stream
        rr = RankRenderer(dist, rank, world, 0, cfg.args(), cfg.dtype, stream, slots=4)
        res = {}
        for scheme in ("fcfs", "cyclic"):
            if rank == 0:
                M.mandel_dev_zero(rr.img, cfg.W * cfg.H * 4, stream)
            dist.barrier()
            st = rr.step(scheme, barrier=True)
            img = None
            if rank == 0:
                host = torch.empty((cfg.H, cfg.W), dtype=torch.int32, pin_memory=True)
                bench._d2h(host, rr.img, cfg.W * cfg.H * 4, stream)
                img = host.numpy().view(np.uint32).copy()
            res[scheme] = (st["kernel"], st["probe"][1], img)
            dist.barrier()
        rr.close()
        q.put((rank, res))
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def test_rank_path_runs_the_view_probe(oracle):
    """mandel_render_rank makes the same per-view EAGER/LAZY choice as mandel_render_ex
    (it always ran batched EAGER, ~0.55x of LAZY on C4): on a C4-like zoom
    every rank process probes on its own device and runs LAZY, and the shared map equals
    the oracle's."""
    cfg = wl.C4.with_(W=1536, H=1536, iter_max=5000)
    want = oracle.render(cfg)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 2
    procs = [ctx.Process(target=_probe_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0, res
    for r in range(world):
        assert isinstance(res[r], dict), res[r]
        for scheme, (kernel, ipe, _) in res[r].items():
            assert kernel == "lazy", (r, scheme, kernel, ipe)
            assert 0 < ipe < 23, (r, scheme, ipe)
    for scheme, (_, _, img) in res[0].items():
        bad = int((img != want).sum())
        assert bad == 0, f"{scheme}: {bad} pixels differ from the oracle"
