"""bench.py's contract on a B200: one JSON line with the keys the driver reads, for the
default single-GPU run and for the one-process-per-GPU path (two ranks sharing the
test box's one GPU through --share-device: the plumbing, not a measurement)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line(out):
    lines = [json.loads(l) for l in out.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, out[-2000:]
    return lines[0]


def _check_contract(d, n_gpus):
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "gpu_launches", "roofline", "clocks",
              "e2e"):
        assert k in d, k
    assert d["metric"] == "pixel-iterations/sec (Giter/s)" and d["unit"] == "Giter/s"
    assert d["value"] > 0 and d["n_gpus"] == n_gpus and d["higher_is_better"] is True
    assert d["dtype"] == "f64" and "workload" in d["config"]
    assert d["gpu_launches"] >= d["steps"]
    r = d["roofline"]
    assert r["bound"] == "alu" and r["unit"] == "TFLOP/s" and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    e = d["e2e"]
    assert e["value"] > 0 and e["unit"] == "Giter/s" and e["d2h_bytes_per_step"] == 4 * d["config"]["pixels"]
    assert e["h2d_bytes_per_step"] == 0 and e["map_sum_check"] is True
    c = d["clocks"]
    assert "sm_mhz" in c and "reasons" in c


def test_bench_single_gpu():
    r = subprocess.run([sys.executable, "bench.py", "--steps", "5", "--warmup", "3", "--e2e-steps", "2",
                        "--no-schemes", "--cpu-seconds", "2"], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _line(r.stdout)
    _check_contract(d, 1)
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["parity_rows_vs_gpu"]["mismatched_pixels"] == 0


@pytest.mark.parametrize("gather,scheme,schemes", [("fused", "fcfs", False), ("nccl", "fcfs", False),
                                                   ("fused", "block", True), ("nccl", "cyclic", True)])
def test_bench_two_ranks_shared_device(gather, scheme, schemes):
    port = {"fused": 29641, "nccl": 29642}[gather] + (10 if schemes else 0)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           "bench.py", "--gpus", "2", "--config", "C1", "--steps", "4", "--warmup", "3",
           "--e2e-steps", "2", "--share-device", "--gather", gather, "--scheme", scheme]
    if not schemes:
        cmd.append("--no-schemes")
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _line(r.stdout)
    _check_contract(d, 2)
    assert d["test_only_shared_device"] is True
    if schemes:
        assert set(d["per_scheme"]) == {"block", "cyclic", "fcfs"}
        assert all(v["value"] > 0 for v in d["per_scheme"].values())
