"""Multi-rank parity cases (TEST CODE) run by tests/mgpu_worker.py, one process
per rank under torchrun: one GPU per rank with NCCL (tests/test_gpu_multi.py),
or all ranks on ONE GPU without NCCL, every exchange over the peer windows
(tests/test_gpu_local_ranks.py).

Every rank runs the pipelined DBP + FWP path through libnest.so; the checks
compare against the CPU oracle over the global batch: routing (uniq /
inverse / masks / count exchange / received keys / owner rows) bit-exact,
pooled rows and tables bit-exact in regime P1 and within 1e-5 in P2
(SURVEY §8(c)).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workload as WL  # noqa: E402
from oracle import cluster as OC  # noqa: E402
from oracle import routing as OR  # noqa: E402
from oracle import step as OS  # noqa: E402


def rel_ok(a, b, tol=1e-5):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.all(np.linalg.norm(a - b, axis=1) <= tol * np.maximum(np.linalg.norm(b, axis=1), 1e-30))


def skewed_batches(cfg, B, T, world, seed=31):
    """Edge case: every key owned by rank 0 (rows multiples of W), and the last
    rank's batch empty (all bags empty) on odd steps."""
    out = []
    for t in range(T):
        per = []
        for r in range(world):
            keys, offs = WL.gen_batch(cfg, seed, t, r, batch=B)
            if r == world - 1 and t % 2 == 1:
                keys, offs = keys[:0], np.zeros_like(offs)
            else:
                tab, row = WL.unpack_keys(keys)
                row = (row // world) * world
                keys = WL.pack_keys(tab, row)
            per.append((keys, offs))
        out.append(per)
    return out


class Case:
    def __init__(self, name, cfg, B, N, T, init, dmode, lr, gen=None, adagrad=None, tables="hbm",
                 schedule="sequential"):
        self.name, self.cfg, self.B, self.N, self.T = name, cfg, B, N, T
        self.init, self.dmode, self.lr, self.gen = init, dmode, lr, gen
        self.adagrad, self.tables, self.schedule = adagrad, tables, schedule

    def inputs(self, world):
        cfg, B, T = self.cfg, self.B, self.T
        F, d = cfg.num_features, cfg.dim
        batches = self.gen(cfg, B, T, world) if self.gen else \
            [[WL.gen_batch(cfg, 21, t, r, batch=B) for r in range(world)] for t in range(T)]
        douts = [[WL.gen_dout(21, t, r, B * F, d, self.dmode) for r in range(world)] for t in range(T)]
        return batches, douts


def overlap_batches(cfg, B, T, world, p_reuse=0.7, seed=41):
    """DBP stress at W > 1: each rank's batch t+1 reuses batch t's key at the
    same slot with probability p_reuse (BASELINE configs[3]), so the refresh /
    re-push (and the early push leaving the pending update's rows to it) carry
    a large intersection."""
    c = cfg.with_(batch_local=B)
    per = [WL.gen_overlap_batches(c, seed, T, r, p_reuse) for r in range(world)]
    return [[per[r][t] for r in range(world)] for t in range(T)]


def cases(big=True):
    out = [
        Case("tiny-P1-N2", WL.CONFIGS["tiny"], 32, 2, 6, "dyadic", "dyadic", 2.0 ** -10),
        Case("tiny-P1-N1", WL.CONFIGS["tiny"], 32, 1, 4, "dyadic", "dyadic", 2.0 ** -10),
        Case("edge-owner0-empty-P1-N2", WL.CONFIGS["tiny"].with_(bag_repeats=True, table_rows=(4000, 800, 64, 9)),
             64, 2, 5, "dyadic", "dyadic", 2.0 ** -10, gen=skewed_batches),
        # clustered FWP schedule across ranks
        Case("tiny-P1-N4-clustered", WL.CONFIGS["tiny"].with_(table_rows=(300, 200, 100, 50), bag_repeats=True),
             64, 4, 4, "dyadic", "dyadic", 2.0 ** -10, schedule="clustered"),
        # row-wise AdaGrad (NEXT-2): (grad_scale, lr, eps), P2 tolerance
        Case("adagrad-P2-N2", WL.CONFIGS["tiny"].with_(table_rows=(3000, 700, 90, 20), zipf=1.2,
                                                       bag_repeats=True, dim=32),
             128, 2, 4, "uniform", "realistic", 0.0, adagrad=(1.0 / 256, 0.05, 1e-8)),
        # soak: many pipelined steps (slot reuse, epoch flags, window reuse)
        Case("soak-P1-N2-40steps", WL.CONFIGS["tiny"].with_(table_rows=(500, 300, 200, 100), bag_repeats=True),
             64, 2, 40, "dyadic", "dyadic", 2.0 ** -12),
        # host-DRAM tier (NEXT-3): every owner's shard in pinned host memory
        Case("host-tier-P1-N2", WL.CONFIGS["tiny"].with_(table_rows=(3000, 40, 7, 999), zipf=1.3,
                                                         bag_repeats=True, dim=128),
             512, 2, 3, "dyadic", "dyadic", 2.0 ** -12, tables="host"),
    ]
    if big:
        out += [
            Case("skew-P1-N4", WL.CONFIGS["tiny"].with_(table_rows=(3000, 40, 7, 999), zipf=1.4, bag_repeats=True,
                                                        dim=128), 1024, 4, 3, "dyadic", "dyadic", 2.0 ** -12),
            Case("mid-P2-N4", WL.CONFIGS["tiny"].with_(table_rows=(20000, 5000, 333, 100000), zipf=1.1,
                                                       bag_repeats=True, dim=64), 2048, 4, 4, "uniform",
                 "realistic", 0.02),
            Case("dbp-overlap-P1-N1", WL.CONFIGS["tiny"].with_(table_rows=(20000, 5000, 3000, 10000), zipf=1.1,
                                                               bag_repeats=True, dim=64),
                 512, 1, 5, "dyadic", "dyadic", 2.0 ** -12, gen=overlap_batches),
        ]
    return out


def make_ctx(case, batches, rank, world, dev, **kw):
    from paper_2604_06956_b200 import NestContext
    cfg = case.cfg
    # one configuration on every rank (the exchange windows must agree)
    Kall = max(1, max(len(b[r][0]) for b in batches for r in range(world)))
    K = Kall
    ada = case.adagrad
    return NestContext(cfg.table_rows, cfg.dim, world=world, rank=rank, max_keys=K, max_batch=case.B,
                       max_micro_batches=case.N, seed=13, init_mode=case.init, device=dev,
                       optimizer="rowwise_adagrad" if ada else "sgd", table_location=case.tables,
                       adagrad_eps=ada[2] if ada else 1e-8,
                       # an owner can receive every rank's keys (edge case: all keys on rank 0)
                       max_recv_keys=world * Kall, max_mb_rows=case.N * K + 64,
                       max_owner_mb_rows=world * case.N * Kall + 64, **kw)


def run_rank(case, ctx, rank, batches, douts, dev, stream=None):
    """The pipelined steps of one rank; returns its pooled rows per step.
    Synchronises only its own streams (other ranks may share the device)."""
    import torch
    from paper_2604_06956_b200.runner import Runner
    F = case.cfg.num_features
    ada = case.adagrad
    with torch.cuda.stream(stream or torch.cuda.current_stream(dev)):
        s = torch.cuda.current_stream(dev)
        run = Runner(ctx, N=case.N, schedule=case.schedule, pipelined=True, lr_over_B=case.lr,
                     adagrad=ada[:2] if ada else None)
        mine = [(torch.from_numpy(b[rank][0]).to(dev), torch.from_numpy(b[rank][1]).to(dev), case.B)
                for b in batches]
        cap = case.B // case.N
        pooled = []
        for t in range(case.T):
            dt = douts[t][rank]
            if case.schedule == "clustered":
                # micro-batch i's gradient rows are its samples' rows (perm order)
                perm, _ = OC.cluster_rounds(OC.sample_keysets(*batches[t][rank], F), case.N)
                dt = dt.reshape(case.B, F, -1)[perm].reshape(case.B * F, -1)
            dd = torch.from_numpy(np.ascontiguousarray(dt)).to(dev)
            outs = run.step(mine[t], mine[t + 1] if t + 1 < case.T else None,
                            lambda tt, i, p, dd=dd: dd[i * cap * F:(i + 1) * cap * F])
            run.join(s)
            s.synchronize()
            pooled.append(np.concatenate([o.cpu().numpy() for o in outs]))
    return pooled


def collect(case, ctx, rank, world, batches, dev):
    """(owned keys, their table rows, route view of the last batch) of one rank."""
    import torch
    allk = np.unique(np.concatenate([b[r][0] for b in batches for r in range(world)]))
    owned = allk[(allk & ((1 << 40) - 1)) % world == rank]
    rows = ctx.read_rows(torch.from_numpy(owned).to(dev)).cpu().numpy()
    view = ctx.route_view((case.T - 1) % 2)
    return owned, rows, {k: v for k, v in view.items() if k != "info"}


def verify(case, world, batches, douts, gathered):
    """gathered[r] = (pooled per step, owned, rows, view) of rank r."""
    cfg, B, N, T = case.cfg, case.B, case.N, case.T
    F, d = cfg.num_features, cfg.dim
    ok = True
    tab = OS.LazyTable(13, d, case.init)
    ada = case.adagrad
    opt = OS.RowwiseAdagrad(lr=ada[1], grad_scale=ada[0], eps=ada[2]) if ada else None
    for t in range(T):
        res = OS.sync_step(tab, batches[t], douts[t], case.lr, optimizer=opt)
        for r in range(world):
            g = gathered[r][0][t]
            # pooled rows come out in micro-batch order (perm), the oracle's in sample order
            ref = res.pooled[r]
            if case.schedule == "clustered":
                ks = OC.sample_keysets(*batches[t][r], F)
                perm, _ = OC.cluster_rounds(ks, N)
                ref = ref.reshape(B, F, d)[perm].reshape(B * F, d)
            good = np.array_equal(g, ref) if case.dmode == "dyadic" else rel_ok(g, ref)
            if not good:
                print(f"[{case.name}] pooled mismatch step {t} rank {r}", flush=True)
                ok = False
    for r in range(world):
        owned_r, rows_r = gathered[r][1], gathered[r][2]
        ref = tab.get(owned_r)
        good = np.array_equal(rows_r, ref) if case.dmode == "dyadic" else rel_ok(rows_r, ref)
        if not good:
            print(f"[{case.name}] table mismatch rank {r}", flush=True)
            ok = False
    # routing of the last batch, bit-exact
    if case.schedule == "clustered":
        sched = [OC.cluster_rounds(OC.sample_keysets(*batches[T - 1][r], F), N) for r in range(world)]
    else:
        sched = [OC.cluster_sequential(B, N)] * world
    mbs = [OR.mb_of_occurrence(batches[T - 1][r][1], F, *sched[r]) for r in range(world)]
    src, own = OR.route_all(batches[T - 1], world, mbs, N)
    for r in range(world):
        v = gathered[r][3]
        checks = {
            "uniq": np.array_equal(v["uniq"], src[r].uniq),
            "inverse": np.array_equal(v["inverse"], src[r].inverse),
            "mask": np.array_equal(v["mask"].astype(np.int64), src[r].mask),
            "send_counts": np.array_equal(v["send_counts"][:, 0], src[r].send_counts)
            and np.array_equal(v["send_counts"][:, 1:1 + N].T, src[r].mb_counts),
            "recv_keys": np.array_equal(v["recv_keys"] & ((1 << 56) - 1), own[r].recv_keys)
            and np.array_equal(v["recv_keys"] >> 56, own[r].recv_mask),
            "owner_inv": np.array_equal(v["owner_inv"], own[r].owner_inv),
        }
        ok_keys = own[r].owner_keys
        tabs, rws = ok_keys >> 40, ok_keys & ((1 << 40) - 1)
        lb = np.concatenate([[0], np.cumsum([(rt - r + world - 1) // world for rt in cfg.table_rows])])
        checks["owner_rows"] = np.array_equal(v["owner_rows"], lb[tabs] + rws // world)
        for s in range(world):
            checks[f"all_counts[{s}]"] = np.array_equal(v["all_counts"][s][:, 0], src[s].send_counts)
        bad = [k for k, good in checks.items() if not good]
        if bad:
            print(f"[{case.name}] routing mismatch rank {r}: {bad}", flush=True)
            ok = False
    print(f"[{case.name}] W={world} {'OK' if ok else 'FAIL'}", flush=True)
    return ok


# ----------------------------------------------------------------------------- trained tower
TOWER = dict(B=32, H=64, lr=0.01)


def tower_ctx(rank, world, dev, **kw):
    from paper_2604_06956_b200 import NestContext
    cfg = WL.CONFIGS["tiny"]
    return NestContext(cfg.table_rows, cfg.dim, world=world, rank=rank, max_keys=TOWER["B"] * cfg.num_features * 3,
                       max_batch=TOWER["B"], seed=2, device=dev, tower_layers=1, tower_hidden=TOWER["H"],
                       tower_train=True, tower_lr=TOWER["lr"], **kw)


def tower_rank(ctx, rank, dev, stream=None):
    """One trained-tower step of one rank: returns (X_r, W0, G, W1)."""
    import torch
    cfg = WL.CONFIGS["tiny"]
    B, F, d = TOWER["B"], cfg.num_features, cfg.dim
    with torch.cuda.stream(stream or torch.cuda.current_stream(dev)):
        s = torch.cuda.current_stream(dev)
        g = torch.Generator(device=dev).manual_seed(100 + rank)
        pooled = (torch.randn((B * F, d), generator=g, device=dev) * 0.5).to(torch.bfloat16)
        dout = torch.empty((B * F, d), dtype=torch.float32, device=dev)
        w0 = ctx.tower_read("weights", 0, stream=s)
        G = ctx.tower_read("top_grad", stream=s)
        ctx.tower_fwd_bwd(pooled, dout, stream=s)
        ctx.tower_step(stream=s)
        ctx.join(s)
        w1 = ctx.tower_read("weights", 0, stream=s)
        s.synchronize()
        return (pooled.float().cpu().numpy(), w0.cpu().double().numpy(), G.cpu().double().numpy()[:B],
                w1.cpu().numpy())


def tower_verify(world, res):
    """NEXT-4: W1 = W0 - lr * sum_r G^T X_r on every rank, bitwise identical replicas."""
    cfg = WL.CONFIGS["tiny"]
    B, F, d, lr = TOWER["B"], cfg.num_features, cfg.dim, TOWER["lr"]
    w0, G = res[0][1], res[0][2]
    Xs = [x.astype(np.float64).reshape(B, F * d) for x, _, _, _ in res]
    ref = w0 - lr * sum(G.T @ X for X in Xs)
    scale = np.abs(w0) + lr * sum(np.abs(G).T @ np.abs(X) for X in Xs)
    ok = all(np.array_equal(res[0][3], r[3]) for r in res) and \
        bool(np.all(np.abs(res[0][3].astype(np.float64) - ref) <= 1e-5 * scale + 1e-7))
    print(f"[tower-train-allreduce] W={world} {'OK' if ok else 'FAIL'}", flush=True)
    return ok
