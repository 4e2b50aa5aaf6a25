"""The N > 1 path of bench.py on a one-GPU box: torchrun with 2 ranks, both on
cuda:0 with gloo collectives (`--functional-1gpu`, a host-logic check, not a
measurement -- the ranks' kernels never wait on one another).  Strong scaling
splits one image over the ranks, so the 2-rank line's NCCL/gloo-summed
checksum and status counts equal the 1-rank line's bit for bit (SURVEY §8(e),
north_star "bit-for-bit reproducible")."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line(cmd):
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("kernel,extra", [("inv_det", ["--rows", "600", "--no-e2e", "--no-extras",
                                                       "--no-cpu-baseline"]),
                                          ("window", ["--rows", "300"])])
def test_two_ranks_equal_one(cuda, kernel, extra):
    common = ["bench.py", "--kernel", kernel, "--steps", "2", "--warmup", "3"] + extra
    one = _line([sys.executable] + common)
    two = _line([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                 "--master-addr", "127.0.0.1", "--master-port", str(_port())] + common +
                ["--gpus", "2", "--functional-1gpu"])
    assert two["n_gpus"] == 2 and one["n_gpus"] == 1
    assert two["checksum"] == one["checksum"]
    if kernel == "inv_det":
        assert two["status_counts"] == one["status_counts"]
        assert sum(two["status_counts"]) == 600 * 40000
