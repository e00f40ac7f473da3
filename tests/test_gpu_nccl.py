"""The NCCL data plane on real hardware: every gpurun call and
the driver's GPU tier get one GPU, so the slab path runs as a one-rank NCCL
group exchanging its axis-0 ghosts with itself (tests/nccl_loopback.py);
fields, diagnostics and host-buffer stepping must equal the one-GPU run
bitwise.  Runs in a subprocess under a timeout so a hung communicator fails
the test instead of stalling the suite."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def test_nccl_loopback_slab_bitwise(built):
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    env.pop("MASTER_PORT", None)
    p = subprocess.run([sys.executable, os.path.join(HERE, "nccl_loopback.py")],
                       capture_output=True, text=True, timeout=600, env=env)
    lines = [json.loads(x) for x in p.stdout.splitlines() if x.startswith("{")]
    bad = [r for r in lines if r.get("ok") is False]
    assert p.returncode == 0 and lines and lines[-1].get("all_ok"), \
        f"rc={p.returncode} failing={bad}\n{p.stdout[-3000:]}\n{p.stderr[-3000:]}"
