"""FWP decomposition, one GPU: the stand-in tower alone
on the full batch vs two half-size calls back to back (no sparse work beside
it), and with one half overlapped by an HBM-bound copy of the pool's size.
Prints ms per step for each."""
import json
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workload as WL  # noqa: E402
from paper_2604_06956_b200 import NestContext  # noqa: E402


def main():
    cfg = WL.CONFIGS["dlrm"]
    B, F, d = cfg.batch_local, cfg.num_features, cfg.dim
    dev = torch.device("cuda", 0)
    ctx = NestContext((1000,) * F, d, num_features=F, max_keys=1024, max_batch=B, seed=1, device=dev,
                      tower_layers=cfg.tower_layers, tower_hidden=cfg.tower_hidden)
    pooled = (torch.randn((B * F, d), device=dev) * 0.1).to(torch.bfloat16)
    dout = torch.empty((B * F, d), device=dev)
    s = torch.cuda.current_stream()

    def run(N, reps=20):
        rows = B * F // N
        for _ in range(3):
            for i in range(N):
                ctx.tower_fwd_bwd(pooled[i * rows:(i + 1) * rows], dout[i * rows:(i + 1) * rows], stream=s)
        ctx.join(s)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            for i in range(N):
                ctx.tower_fwd_bwd(pooled[i * rows:(i + 1) * rows], dout[i * rows:(i + 1) * rows], stream=s)
        ctx.join(s)
        e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    out = {"tower_alone_ms": {f"N{N}": run(N) for N in (1, 2, 4)}}
    flops = 3 * 2 * B * (F * d * cfg.tower_hidden + (cfg.tower_layers - 1) * cfg.tower_hidden ** 2)
    out["tower_tflops"] = {k: flops / (v * 1e9) for k, v in out["tower_alone_ms"].items()}
    print(json.dumps(out))
    ctx.close()


if __name__ == "__main__":
    main()
