"""World-size-2 host-side tests of the multi-rank path over gloo (CPU, -m "not gpu").

Each rank produces its row of the count exchange (the oracle plays the
device's role), the rows are all-gathered over gloo exactly as nest_route
all-gathers them over NCCL, and the product's host planner
(nest_exchange_plan, the code nest_route runs after its host sync) must give
every rank the All2All displacements the oracle's simulated fabric implies
 and take the same capacity decision on every rank.
"""
import ctypes as C
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import workload as WL
        from oracle import cluster as OC
        from oracle import routing as OR
        from paper_2604_06956_b200 import _lib as L
        lib = L.load()
        cfg = WL.CONFIGS["tiny"]
        N, B, Nmax = 2, 32, 4
        Nc = Nmax + 2
        batches = [WL.gen_batch(cfg, 9, 0, r, batch=B) for r in range(world)]
        perm, mbo = OC.cluster_sequential(B, N)
        mbs = [OR.mb_of_occurrence(b[1], cfg.num_features, perm, mbo) for b in batches]
        src, own = OR.route_all(batches, world, mbs, N)
        # this rank's row: per owner {U, U_1..U_N, (unused), err}
        row = np.zeros((world, Nc), dtype=np.int32)
        rs = src[rank]
        for o in range(world):
            row[o, 0] = rs.send_counts[o]
            row[o, 1:1 + N] = rs.mb_counts[:, o]
        gathered = [torch.zeros((world, Nc), dtype=torch.int32) for _ in range(world)]
        dist.all_gather(gathered, torch.from_numpy(row))
        allc = np.ascontiguousarray(torch.stack(gathered).numpy())
        rows = (C.c_int64 * cfg.num_tables)(*cfg.table_rows)

        def conf(max_recv=0):
            return L.Config(world=world, rank=rank, num_tables=cfg.num_tables, dim=cfg.dim, table_rows=rows,
                            pooling=0, num_features=cfg.num_features, max_keys=B * 12, max_batch=B,
                            max_micro_batches=Nmax, max_recv_keys=max_recv, seed=1)
        c0 = conf()
        plan = L.ExchangePlan()
        rc = lib.nest_exchange_plan(C.byref(c0), N, allc.ctypes.data, C.byref(plan))
        assert rc == 0, rc
        ow = own[rank]
        assert plan.uniq == len(rs.uniq)
        assert plan.recv == len(ow.recv_keys)
        assert list(plan.key_send_off[:world + 1]) == list(rs.send_offsets)
        assert list(plan.key_recv_off[:world + 1]) == list(ow.recv_offsets)
        for i in range(N):
            assert plan.mb_uniq[i] == int(((rs.mask >> i) & 1).sum())
            assert plan.mb_recv[i] == sum(len(ow.send_lists[i][s]) for s in range(world))
            assert plan.src_base[i + 1] - plan.src_base[i] == plan.mb_uniq[i]
            assert plan.own_base[i + 1] - plan.own_base[i] == plan.mb_recv[i]
        # shard rows over ranks partition the tables
        sr = torch.tensor([lib.nest_shard_rows(C.byref(c0))], dtype=torch.int64)
        dist.all_reduce(sr)
        assert int(sr.item()) == sum(cfg.table_rows)
        # a capacity violation at ONE owner is decided identically on every rank
        smallest = min(len(o.recv_keys) for o in own)
        largest = max(len(o.recv_keys) for o in own)
        cap = (smallest + largest) // 2 if largest > smallest else largest - 1
        rc2 = lib.nest_exchange_plan(C.byref(conf(cap)), N, allc.ctypes.data, C.byref(plan))
        codes = [torch.zeros(1, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(codes, torch.tensor([rc2], dtype=torch.int32))
        assert all(int(x.item()) == 4 for x in codes), [int(x.item()) for x in codes]
        # an error flag raised by any rank reaches every rank's decision
        bad = allc.copy()
        bad[1, 0, Nc - 1] = 1
        rc3 = lib.nest_exchange_plan(C.byref(c0), N, bad.ctypes.data, C.byref(plan))
        assert rc3 == 5
        q.put((rank, "ok"))
    except BaseException as e:  # pragma: no cover
        import traceback
        q.put((rank, "".join(traceback.format_exception(e))))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_exchange_plan():
    import torch.multiprocessing as mp
    from paper_2604_06956_b200 import build as B
    B.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
