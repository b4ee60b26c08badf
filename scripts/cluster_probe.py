"""Times one GPU clustering (B=65,536, DLRM keys) -- used under ncu for the
per-kernel launch list."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workload as WL
from paper_2604_06956_b200 import NestContext
cfg = WL.CONFIGS["dlrm"]
N = int(sys.argv[1]) if len(sys.argv) > 1 else 4
if len(sys.argv) > 2:
    cfg = cfg.with_(zipf=float(sys.argv[2]))
W = int(sys.argv[3]) if len(sys.argv) > 3 else 1
keys, offs = WL.gen_batch(cfg, 0, 0, 0)
dev = torch.device("cuda:0")
ctx = NestContext(cfg.table_rows, cfg.dim, max_keys=len(keys), max_batch=cfg.batch_local,
                  max_micro_batches=max(N, 2), init_tables=False, device=dev)
side = torch.cuda.Stream()
kd, od = torch.from_numpy(keys).to(dev), torch.from_numpy(offs).to(dev)
for rep in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    with torch.cuda.stream(side):
        perm, mbo = ctx.fwp_schedule(kd, od, cfg.batch_local, N, "clustered", stream=side)
    torch.cuda.synchronize()
    p = perm.cpu().numpy()
    assert sorted(p.tolist()) == list(range(cfg.batch_local)), "perm is not a permutation"
    e1.record()
    torch.cuda.synchronize()
    print(f"N={N} clustered schedule: {e0.elapsed_time(e1):.3f} ms")
