"""Multi-GPU parity through real NCCL (needs >= 2 GPUs; -m gpu)."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ndev():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


# transports: fused NVLink stores with the early push (default), fused with
# the embedding push inside the window, copy engines, NCCL send/recv
TRANSPORTS = {"fused-early": {}, "fused-early-ce": {"NEST_EARLY_PUSH": "ce"},
              "fused-early-gradce": {"NEST_GRAD_PUSH": "ce"},
              "fused-early-range": {"NEST_SEGSUM": "range"},
              "fused-window": {"NEST_EARLY_PUSH": "0"}, "ce": {"NEST_A2A": "ce"},
              "nccl": {"NEST_A2A": "nccl"},
              # count exchange + key All2All over the windows too (no NCCL on the route)
              # count exchange + key All2All over NCCL (the default puts them on the windows)
              "fused-early-routenccl": {"NEST_ROUTE_XCHG": "nccl"},
              # no NCCL at all: windows connected through torch.distributed
              "no-nccl": {"NEST_MGPU_NO_NCCL": "1"},
              # every key's gradient row to its owner (no direct write-back)
              "fused-early-nodwb": {"NEST_DIRECT_WB": "0"}}


@pytest.mark.parametrize("world,transport", [(2, t) for t in TRANSPORTS] +
                         [(4, "fused-early"), (4, "no-nccl"), (8, "fused-early"), (8, "no-nccl")])
def test_multi_rank_parity(world, transport):
    if _ndev() < world:
        pytest.skip(f"needs >= {world} CUDA devices")
    def cmd():
        return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
                "--master-addr", "127.0.0.1", "--master-port", str(_port()),
                os.path.join(ROOT, "tests", "mgpu_worker.py")]
    env = dict(os.environ, **TRANSPORTS[transport])
    for _ in range(3):   # a free port can be taken between probing and torchrun binding it
        r = subprocess.run(cmd(), cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
        if "EADDRINUSE" not in r.stderr:
            break
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0 and "MGPU ALL OK" in r.stdout
