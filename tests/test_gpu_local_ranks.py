"""Multi-rank parity on ONE GPU (-m gpu): W = 2, 4, 8 ranks as W processes
sharing cuda:0 (tests/mgpu_worker.py with NEST_MGPU_SAME_DEVICE=1), no NCCL:
every exchange runs over the peer windows (CUDA IPC on the same device).  This
runs the W > 1 rows of SURVEY §8(a) -- R2 count exchange + key All2All, R3
owner dedup, R6 owner send gather, R7 embedding All2All, R10 segment-sum into
the owners' rows, R11 gradient All2All, R12 owner reduce + update -- and the
trained tower's AllReduce (NEXT-4) on a single-GPU box, against the oracle.
The kernels are the multi-GPU kernels; only where the peers' windows live
differs.  Launched with a timeout, so a stuck exchange cannot hang the suite."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# transports of the row exchanges (R7 / R11): fused stores with the early push
# (default), copy engines, the range segment-sum at W > 1, pushes inside the
# window, the copy-engine early push
TRANSPORTS = {"fused-early": {}, "ce": {"NEST_A2A": "ce"}, "fused-range": {"NEST_SEGSUM": "range"},
              "fused-window": {"NEST_EARLY_PUSH": "0"}, "fused-early-ce": {"NEST_EARLY_PUSH": "ce"},
              # checked mode: guard bands after every workspace buffer verified after each case
              "fused-early-guard": {"NEST_GUARD": "1"},
              # zero-copy retrieval: owners push / update their shard rows in place
              "fused-early-zerocopy": {"NEST_ZERO_COPY": "1"},
              # every key's gradient row goes to its owner (no direct write-back)
              "fused-early-nodwb": {"NEST_DIRECT_WB": "0"}}


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,transport,big", [(2, "fused-early", True), (4, "fused-early", False),
                                                 (8, "fused-early", False), (2, "ce", False),
                                                 (4, "fused-range", False), (2, "fused-window", False),
                                                 (2, "fused-early-ce", False), (4, "fused-early-guard", False),
                                                 (2, "fused-early-zerocopy", True), (4, "fused-early-zerocopy", False),
                                                 (2, "fused-early-nodwb", True)])
def test_local_ranks_parity(world, transport, big):
    def cmd():
        return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
                "--master-addr", "127.0.0.1", "--master-port", str(_port()),
                os.path.join(ROOT, "tests", "mgpu_worker.py")]
    env = dict(os.environ, NEST_MGPU_SAME_DEVICE="1", NEST_MGPU_BIG="1" if big else "0",
               **TRANSPORTS[transport])
    for _ in range(3):   # a free port can be taken between probing and torchrun binding it
        r = subprocess.run(cmd(), cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
        if "EADDRINUSE" not in r.stderr:
            break
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0 and "MGPU ALL OK" in r.stdout
    # the direct write-back runs wherever it applies (fused SM pushes, SGD, HBM)
    dwb = "direct write-back on" in r.stdout
    assert dwb == (transport not in ("ce", "fused-early-ce", "fused-early-nodwb")), "direct write-back state"
