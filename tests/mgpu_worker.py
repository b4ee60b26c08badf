"""Multi-rank parity worker (launched by torchrun; tests/test_gpu_multi.py and
tests/test_gpu_local_ranks.py).

One process per rank.  Default: one GPU per rank with real NCCL.
NEST_MGPU_NO_NCCL=1: no NCCL -- the exchange windows are connected through
torch.distributed and every exchange of the path runs over them.
NEST_MGPU_SAME_DEVICE=1 (implies no NCCL): every rank on cuda:0, the process
group on gloo -- W ranks on ONE GPU, each process its own CUDA context (own
hardware queues, time-sliced), the peers' windows mapped through CUDA IPC on
the same device: the W > 1 kernels and exchanges run on a single-GPU box.  The cases and checks are tests/multirank.py's: rank 0 compares
against the CPU oracle over the global batch -- routing bit-exact, pooled rows
and tables bit-exact in regime P1 and within 1e-5 in P2.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import multirank as MR  # noqa: E402
from paper_2604_06956_b200 import unique_ids  # noqa: E402
from paper_2604_06956_b200._lib import WindowRec  # noqa: E402

SAME_DEVICE = os.environ.get("NEST_MGPU_SAME_DEVICE", "0") == "1"
NO_NCCL = SAME_DEVICE or os.environ.get("NEST_MGPU_NO_NCCL", "0") == "1"


def flag_tensor(ok, dev):
    return torch.tensor([1 if ok else 0], device="cpu" if SAME_DEVICE else dev)


def ctx_kw(rank):
    if NO_NCCL:
        return {}
    obj = [unique_ids() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return {"nccl_uids": obj[0]}


def connect(ctx, world):
    if NO_NCCL:
        recs = [None] * world
        mine = ctx.window_export()
        dist.all_gather_object(recs, mine)
        ctx.window_connect(recs)
        # direct write-back of sole-contributor keys (fused transport, SGD, HBM):
        # this rank exported its shard for the peers' write-backs
        rec = WindowRec.from_buffer_copy(mine)
        print(f"[window] rank {dist.get_rank()}: direct write-back {'on' if rec.dwb_ok else 'off'}", flush=True)


def run_case(case, rank, world, dev):
    batches, douts = case.inputs(world)
    ctx = MR.make_ctx(case, batches, rank, world, dev, **ctx_kw(rank))
    connect(ctx, world)
    pooled = MR.run_rank(case, ctx, rank, batches, douts, dev)
    res = (pooled,) + MR.collect(case, ctx, rank, world, batches, dev)
    guard_ok = True
    if os.environ.get("NEST_GUARD") == "1":   # checked mode: no out-of-bounds workspace write
        bad = ctx.check_guards()
        guard_ok = bad == 0
        print(f"[{case.name}] rank {rank}: guard bands {'intact' if guard_ok else f'{bad} words overwritten'}",
              flush=True)
    gathered = [None] * world if rank == 0 else None
    dist.gather_object(res, gathered, dst=0)
    ok = MR.verify(case, world, batches, douts, gathered) if rank == 0 else True
    ctx.close()
    flag = flag_tensor(ok and guard_ok, dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    return bool(flag.item())


def run_tower(rank, world, dev):
    ctx = MR.tower_ctx(rank, world, dev, **ctx_kw(rank))
    connect(ctx, world)
    res = MR.tower_rank(ctx, rank, dev)
    gathered = [None] * world if rank == 0 else None
    dist.gather_object(res, gathered, dst=0)
    ok = MR.tower_verify(world, gathered) if rank == 0 else True
    ctx.close()
    flag = flag_tensor(ok, dev)
    dist.broadcast(flag, 0)
    return bool(flag.item())


def main():
    if os.environ.get("NEST_MGPU_DUMP_AFTER"):
        # debugging aid: dump every thread's stack (and exit) if a rank is stuck
        import faulthandler
        faulthandler.dump_traceback_later(int(os.environ["NEST_MGPU_DUMP_AFTER"]), exit=True)
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = 0 if SAME_DEVICE else int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if SAME_DEVICE:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=dev)
    all_ok = run_tower(rank, world, dev)
    only = os.environ.get("NEST_MGPU_ONLY", "")
    big = os.environ.get("NEST_MGPU_BIG", "1") == "1"
    for case in MR.cases(big=big):
        if only and only not in case.name:
            continue
        all_ok &= run_case(case, rank, world, dev)
    if SAME_DEVICE:
        dist.barrier()
    else:
        dist.barrier(device_ids=[local])
    dist.destroy_process_group()
    if rank == 0:
        print("MGPU ALL OK" if all_ok else "MGPU FAILED", flush=True)
    sys.exit(0 if all_ok else 1)


if __name__ == "__main__":
    main()
