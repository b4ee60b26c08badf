"""NVLink anchor for the row All2All: torch.distributed.all_to_all_single (NCCL)
of fp32 rows, equal splits, on the same box as the bench (run under torchrun).
Prints per-GPU algbw (bytes each GPU sends off-GPU / time) and NCCL busbw."""
import json
import os

import torch
import torch.distributed as dist


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    out = {}
    for mb in (64, 256, 600):
        n = (mb << 20) // 4 // world * world
        x = torch.randn(n, device="cuda")
        y = torch.empty_like(x)
        for _ in range(3):
            dist.all_to_all_single(y, x)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        it = 20
        e0.record()
        for _ in range(it):
            dist.all_to_all_single(y, x)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / it
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        off = 4 * n * (world - 1) / world       # bytes each GPU sends to its peers
        out[f"{mb}MB"] = {"ms": ms, "offgpu_gbs_per_gpu": off / (ms * 1e6),
                          "busbw_gbs": (4 * n / (ms * 1e6)) * (world - 1) / world}
    if rank == 0:
        print(json.dumps({"world": world, "nccl_all_to_all_single": out}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
