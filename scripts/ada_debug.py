"""Debug: row-wise AdaGrad W=1 N=1 pipelined vs oracle -- worst rows per form."""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import workload as WL
from oracle import step as OS
from paper_2604_06956_b200 import NestContext
from paper_2604_06956_b200.runner import Runner

DEV = torch.device("cuda:0")
N, pipelined = int(sys.argv[1]), sys.argv[2] == "1"
cfg = WL.CONFIGS["tiny"].with_(table_rows=(5000, 3000, 200, 77), zipf=1.3, bag_repeats=True, dim=32)
B, T, F, d, seed = 256, 5, cfg.num_features, cfg.dim, 7
batches = [[WL.gen_batch(cfg, seed, t, 0, batch=B)] for t in range(T)]
douts = [[WL.gen_dout(seed, t, 0, B * F, d, "realistic")] for t in range(T)]
K = max(len(b[0][0]) for b in batches)
gs, lr, eps = 1.0 / B, 0.05, 1e-8
res = []
for rep in range(2):
    ctx = NestContext(cfg.table_rows, d, pooling=cfg.pooling, max_keys=K, max_batch=B, max_micro_batches=N, seed=11,
                      init_mode="uniform", device=DEV, optimizer="rowwise_adagrad", adagrad_eps=eps)
    run = Runner(ctx, N=N, pipelined=pipelined, adagrad=(gs, lr))
    dev_b = [(torch.from_numpy(b[0][0]).to(DEV), torch.from_numpy(b[0][1]).to(DEV), B) for b in batches]
    cap = B // N
    dds = [torch.from_numpy(douts[t][0]).to(DEV) for t in range(T)]
    for t in range(T):
        run.step(dev_b[t], dev_b[t + 1] if t + 1 < T else None, lambda tt, i, p, dd=dds[t]: dd[i * cap * F:(i + 1) * cap * F])
    run.join()
    torch.cuda.synchronize()
    allk = np.unique(np.concatenate([b[0][0] for b in batches]))
    kd = torch.from_numpy(allk).to(DEV)
    res.append((ctx.read_rows(kd).cpu().numpy(), ctx.read_state(kd).cpu().numpy()))
    ctx.close()
tab = OS.LazyTable(11, d, "uniform")
opt = OS.RowwiseAdagrad(lr=lr, grad_scale=gs, eps=eps)
for t in range(T):
    OS.sync_step(tab, batches[t], douts[t], 0.0, optimizer=opt)
ref = tab.get(allk)
refm = opt.get_state(allk)
got, m = res[0]
err = np.linalg.norm(got - ref, axis=1) / np.linalg.norm(ref, axis=1)
merr = np.abs(m - refm) / refm
cnt = {k: 0 for k in allk}
for b in batches:
    for k in b[0][0]:
        cnt[k] += 1
o = np.argsort(-err)[:5]
print(os.environ.get("NEST_SEGSUM", "default"), "N", N, "pipe", pipelined, "deterministic", np.array_equal(res[0][0], res[1][0]),
      "max row err", err.max(), "worst keys", [(int(allk[i]), float(err[i]), cnt[allk[i]], float(merr[i])) for i in o])
