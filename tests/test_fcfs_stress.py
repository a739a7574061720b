"""FCFS under injected delays: the claim protocol of the library's
kernels -- one atomic per chunk on the shared counter, each chunk bound one chunk
ahead, ranks that never wait on one another -- run with random sleeps before every
claim, between a claim and its visible binding, at warp start and before stores
(libmandel_delay.so), for N in {2, 3, 5, 8} logical ranks x {FCFS, FCFS_MASTER} (and the
single claimant's 16-chunk batches, FCFS at N = 1) x 20 repetitions on a 64x64 and a C1-class view.  Every map equals the oracle's and every
chunk is claimed exactly once."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_fcfs_claims_under_injected_delays():
    from paper_2007_00745_b200 import build
    lib = build.build_delay()
    env = dict(os.environ, MANDEL_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "fcfs_delay_stress.py"), "--reps", "20"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-3000:])
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["library"] == "libmandel_delay.so"
    assert d["mismatched_renders"] == 0 and d["renders"] == 2 * (2 * 4 + 1) * 20
