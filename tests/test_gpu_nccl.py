"""The N > 1 exchanges over real NCCL on one GPU: a single-rank process group
with every collective of the sharded iteration forced on (tests/nccl_single_rank.py);
the trace must equal the shortcut (no-collective) run bit for bit. The
multi-rank arithmetic itself is covered with gloo at world sizes 2 and 4
(tests/test_dist_gloo.py)."""
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
HELPER = Path(__file__).resolve().parent / "nccl_single_rank.py"


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("name,iters", [("water@s24", 3), ("source64@s24", 2)])
def test_nccl_collectives_single_rank(name, iters):
    env = {"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(_port()), "PATH": "/usr/bin:/bin"}
    import os

    env = {**os.environ, **env}
    r = subprocess.run([sys.executable, str(HELPER), name, str(iters)], capture_output=True, text=True, timeout=600,
                       env=env)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
