"""Multi-GPU parity worker (launched by torchrun; see tests/test_gpu_multi.py).

Every rank runs the pipelined DBP + FWP path through libnest.so with real NCCL
All2Alls; rank 0 compares against the CPU oracle over the global batch:
routing (uniq / inverse / masks / count exchange / received keys / owner rows)
bit-exact, pooled rows and tables bit-exact in regime P1 and within 1e-5 in P2.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import workload as WL  # noqa: E402
from oracle import cluster as OC  # noqa: E402
from oracle import routing as OR  # noqa: E402
from oracle import step as OS  # noqa: E402
from paper_2604_06956_b200 import NestContext, unique_ids  # noqa: E402
from paper_2604_06956_b200.runner import Runner  # noqa: E402


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


def tower_case(rank, world, dev):
    """NEXT-4: the trained tower's dense gradients are summed over the ranks
    (AllReduce) before the SGD step: W1 = W0 - lr * sum_r G^T X_r on every
    rank, bitwise identical replicas."""
    cfg = WL.CONFIGS["tiny"]
    B, F, d, H, lr = 32, cfg.num_features, cfg.dim, 64, 0.01
    obj = [unique_ids() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ctx = NestContext(cfg.table_rows, d, world=world, rank=rank, max_keys=B * F * 3, max_batch=B,
                      seed=2, nccl_uids=obj[0], device=dev, tower_layers=1, tower_hidden=H, tower_train=True,
                      tower_lr=lr)
    g = torch.Generator(device=dev).manual_seed(100 + rank)
    pooled = (torch.randn((B * F, d), generator=g, device=dev) * 0.5).to(torch.bfloat16)
    dout = torch.empty((B * F, d), dtype=torch.float32, device=dev)
    w0 = ctx.tower_read("weights", 0).cpu().double().numpy()
    G = ctx.tower_read("top_grad").cpu().double().numpy()[:B]
    ctx.tower_fwd_bwd(pooled, dout)
    ctx.tower_step()
    ctx.join()
    torch.cuda.synchronize()
    w1 = ctx.tower_read("weights", 0).cpu().numpy()
    xs = [None] * world if rank == 0 else None
    dist.gather_object((pooled.float().cpu().numpy(), w1), xs, dst=0)
    ok = True
    if rank == 0:
        Xs = [x.astype(np.float64).reshape(B, F * d) for x, _ in xs]
        ref = w0 - lr * sum(G.T @ X for X in Xs)
        scale = np.abs(w0) + lr * sum(np.abs(G).T @ np.abs(X) for X in Xs)
        ok = all(np.array_equal(xs[0][1], w) for _, w in xs) and \
            bool(np.all(np.abs(xs[0][1].astype(np.float64) - ref) <= 1e-5 * scale + 1e-7))
        print(f"[tower-train-allreduce] {'OK' if ok else 'FAIL'}", flush=True)
    ctx.close()
    return ok


def run_case(name, cfg, B, N, T, init, dmode, lr, rank, world, dev, uids, gen=None, adagrad=None,
             tables="hbm"):
    F, d = cfg.num_features, cfg.dim
    batches = gen(cfg, B, T, world) if gen else \
        [[WL.gen_batch(cfg, 21, t, r, batch=B) for r in range(world)] for t in range(T)]
    douts = [[WL.gen_dout(21, t, r, B * F, d, dmode) for r in range(world)] for t in range(T)]
    K = max(1, max(len(b[rank][0]) for b in batches))
    ctx = NestContext(cfg.table_rows, d, world=world, rank=rank, max_keys=K, max_batch=B,
                      max_micro_batches=N, seed=13, init_mode=init, nccl_uids=uids, device=dev,
                      optimizer="rowwise_adagrad" if adagrad else "sgd", table_location=tables,
                      adagrad_eps=adagrad[2] if adagrad else 1e-8)
    run = Runner(ctx, N=N, pipelined=True, lr_over_B=lr, adagrad=adagrad[:2] if adagrad else None)
    mine = [(torch.from_numpy(b[rank][0]).to(dev), torch.from_numpy(b[rank][1]).to(dev), B) for b in batches]
    cap = B // N
    pooled = []
    for t in range(T):
        dd = torch.from_numpy(douts[t][rank]).to(dev)
        outs = run.step(mine[t], mine[t + 1] if t + 1 < T else None,
                        lambda tt, i, p, dd=dd: dd[i * cap * F:(i + 1) * cap * F])
        torch.cuda.synchronize()
        pooled.append(np.concatenate([o.cpu().numpy() for o in outs]))
    # route view of the last batch
    view = ctx.route_view((T - 1) % 2)
    allk = np.unique(np.concatenate([b[r][0] for b in batches for r in range(world)]))
    owned = allk[(allk & ((1 << 40) - 1)) % world == rank]
    rows = ctx.read_rows(torch.from_numpy(owned).to(dev)).cpu().numpy()
    gathered = [None] * world if rank == 0 else None
    dist.gather_object((pooled, owned, rows, {k: v for k, v in view.items() if k != "info"}), gathered, dst=0)
    ok = True
    if rank == 0:
        tab = OS.LazyTable(13, d, init)
        opt = OS.RowwiseAdagrad(lr=adagrad[1], grad_scale=adagrad[0], eps=adagrad[2]) if adagrad else None
        for t in range(T):
            res = OS.sync_step(tab, batches[t], douts[t], lr, optimizer=opt)
            for r in range(world):
                g = gathered[r][0][t]
                good = np.array_equal(g, res.pooled[r]) if dmode == "dyadic" else rel_ok(g, res.pooled[r])
                if not good:
                    print(f"[{name}] pooled mismatch step {t} rank {r}", flush=True)
                    ok = False
        for r in range(world):
            owned_r, rows_r = gathered[r][1], gathered[r][2]
            ref = tab.get(owned_r)
            good = np.array_equal(rows_r, ref) if dmode == "dyadic" else rel_ok(rows_r, ref)
            if not good:
                print(f"[{name}] table mismatch rank {r}", flush=True)
                ok = False
        # routing of the last batch, bit-exact
        perm, mbo = OC.cluster_sequential(B, N)
        mbs = [OR.mb_of_occurrence(batches[T - 1][r][1], F, perm, mbo) for r in range(world)]
        src, own = OR.route_all(batches[T - 1], world, mbs, N)
        Nc = N + 2
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
                print(f"[{name}] routing mismatch rank {r}: {bad}", flush=True)
                ok = False
        print(f"[{name}] {'OK' if ok else 'FAIL'}", flush=True)
    ctx.close()
    flag = torch.tensor([1 if ok else 0], device=dev)
    dist.broadcast(flag, 0)
    return bool(flag.item())


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    cases = [
        ("tiny-P1-N2", WL.CONFIGS["tiny"], 32, 2, 6, "dyadic", "dyadic", 2.0 ** -10),
        ("tiny-P1-N1", WL.CONFIGS["tiny"], 32, 1, 4, "dyadic", "dyadic", 2.0 ** -10),
        ("skew-P1-N4", WL.CONFIGS["tiny"].with_(table_rows=(3000, 40, 7, 999), zipf=1.4, bag_repeats=True,
                                                 dim=128), 1024, 4, 3, "dyadic", "dyadic", 2.0 ** -12),
        ("mid-P2-N4", WL.CONFIGS["tiny"].with_(table_rows=(20000, 5000, 333, 100000), zipf=1.1,
                                                bag_repeats=True, dim=64), 2048, 4, 4, "uniform",
         "realistic", 0.02),
    ]
    # (name, cfg, B, N, T, init, dout mode, lr, batch generator)
    cases.append(("edge-owner0-empty-P1-N2", WL.CONFIGS["tiny"].with_(bag_repeats=True, table_rows=(4000, 800, 64, 9)),
                  64, 2, 5, "dyadic", "dyadic", 2.0 ** -10, skewed_batches))
    # row-wise AdaGrad (NEXT-2): (grad_scale, lr, eps), P2 tolerance
    cases.append(("adagrad-P2-N2", WL.CONFIGS["tiny"].with_(table_rows=(3000, 700, 90, 20), zipf=1.2,
                                                            bag_repeats=True, dim=32),
                  128, 2, 4, "uniform", "realistic", 0.0, None, (1.0 / 256, 0.05, 1e-8)))
    # host-DRAM tier (NEXT-3): every owner's shard in pinned host memory
    cases.append(("host-tier-P1-N2", WL.CONFIGS["tiny"].with_(table_rows=(3000, 40, 7, 999), zipf=1.3,
                                                              bag_repeats=True, dim=128),
                  512, 2, 3, "dyadic", "dyadic", 2.0 ** -12, None, None, "host"))
    all_ok = True
    all_ok &= tower_case(rank, world, dev)
    for case in cases:
        obj = [unique_ids() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        gen = case[8] if len(case) > 8 else None
        ada = case[9] if len(case) > 9 else None
        tables = case[10] if len(case) > 10 else "hbm"
        all_ok &= run_case(*case[:8], rank, world, dev, obj[0], gen=gen, adagrad=ada, tables=tables)
    dist.barrier(device_ids=[local])
    dist.destroy_process_group()
    if rank == 0:
        print("MGPU ALL OK" if all_ok else "MGPU FAILED", flush=True)
    sys.exit(0 if all_ok else 1)


if __name__ == "__main__":
    main()
