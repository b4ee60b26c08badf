#!/usr/bin/env python
"""Embedding-step benchmark (BASELINE.json metric) for the NestPipe hot path.

One step = the whole hot path of SURVEY.md §8(a) over one batch per GPU:
FWP schedule, DBP route of the next batch (dedup, count exchange, key
All2All, owner dedup, prefetch gather), the frozen window of N micro-batches
(send gather, embedding All2All, pool, segment-sum, gradient All2All), the
fused owner reduce + SGD + write-back, and the dual-buffer refresh.  Weak
scaling: 65,536 samples per GPU, fixed tables.

The headline `value` is the step with the stand-in dense tower as FWP's
overlap partner (variant E+T; north_star: "the overlap partner, not the
product"; its scaling target is "with FWP hiding most All2All behind dense
compute").  Also reported: the same step at the other micro-batch count
(`fwp.with_tower`: exposed All2All without / with FWP) and the embedding
step alone (`embedding_only`, variant E: the loss gradient of the pooled rows
is a fixed tensor).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Rank 0 prints ONE JSON line.  `--impl reference` times the CPU oracle (this
tier's reference arm) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workload as WL  # noqa: E402

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
UNIT = "samples/s"
NVLINK_PEER_GBS = 770.0    # measured peer copy per direction (B200_PROFILING.md)
NVLINK_NOMINAL_GBS = 900.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)   # >= 10 warm-up, >= 50 timed
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="dlrm", choices=["dlrm", "tiny", "dbp_stress", "genrec"])
    ap.add_argument("--zipf", type=float, default=0.0, help="override the config's Zipf skew (FWP sweep)")
    ap.add_argument("--reuse", type=float, default=0.0,
                    help="DBP stress: batch t+1 reuses each key slot of batch t with this probability")
    ap.add_argument("--correlated", default="", help="G,rho: correlated sample groups (FWP clustering sweep)")
    ap.add_argument("--micro-batches", type=int, default=0,
                    help="FWP micro-batches N; 0 = auto (1; N = 2 is measured alongside)")
    ap.add_argument("--schedule", default="sequential", choices=["sequential", "clustered", "clustered-offline"],
                    help="FWP partition: sequential, clustered (GPU greedy per batch, timed), "
                         "clustered-offline (P:482: computed once per batch outside the step, cost reported)")
    ap.add_argument("--variant", default="et", choices=["et", "e"],
                    help="et: embedding + stand-in tower (FWP overlap partner; headline); e: embedding only")
    ap.add_argument("--batches", type=int, default=3, help="distinct batches cycled per rank")
    ap.add_argument("--optimizer", default="sgd", choices=["sgd", "rowwise_adagrad"],
                    help="sparse update: SGD of Eq. 2 (default) or row-wise AdaGrad (SURVEY NEXT-2)")
    ap.add_argument("--tables", default="hbm", choices=["hbm", "host"],
                    help="table tier: HBM (default) or pinned host DRAM over PCIe (SURVEY NEXT-3)")
    ap.add_argument("--tower-layers", type=int, default=0,
                    help="stand-in tower depth L (0: the config's, 4); the FWP sweep runs L in {2, 4, 8} (P:832-835)")
    ap.add_argument("--tower-train", action="store_true",
                    help="train the stand-in tower: dense dW AllReduce + SGD on the dW stream (SURVEY NEXT-4)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--seeds", type=int, default=1,
                    help="SURVEY §8(d) protocol: time the step on the batches of seeds seed..seed+n-1 "
                         "(one context, re-routed per seed) and report the median step time")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fwp-compare", action="store_true",
                    help="skip the secondary runs (other micro-batch count, other variant)")
    ap.add_argument("--trace", default="", help="write the per-stage trace JSON here")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d.get("hbm_gbs", 6650.0)), float(d.get("bf16_tflops_sustained", 1400.0)), "measured"
    return 6650.0, 1400.0, "fallback"


HBM_STAGES = ["route", "sort", "owner_dedup", "gather", "refresh", "send_gather", "pool", "segsum", "update",
              "emb_repush"]
# fused transport stages (W > 1, or W = 1 with micro-batches): their `bytes` are
# off-GPU bytes; their local-HBM bytes (rows gathered / the segment-sum's reads
# + rows stored locally) come in `hbm_bytes`
XFER_STAGES = ["key_a2a", "emb_a2a", "grad_a2a"]


def whole_step_hbm(st, steps, ms_step):
    """Algorithmic HBM bytes of every stage of the step (SURVEY §8(d) per-kernel
    formulas, summed) over the step time, against the measured copy peak."""
    hbm_peak, _, src = peaks()
    used = [n for n in HBM_STAGES + XFER_STAGES if n in st and st[n]["records"]
            and (n in HBM_STAGES or st[n].get("hbm_bytes", 0.0) > 0)]
    b = sum(st[n]["bytes"] if n in HBM_STAGES else st[n]["hbm_bytes"] for n in used) / steps
    gbs = b / (ms_step * 1e6)
    return {"bytes_per_step": b, "gbs": gbs, "peak": hbm_peak, "frac": gbs / hbm_peak, "peak_source": src,
            "stages": used}


def roofline_from(st, key_prefix):
    """HBM roofline of the dominant single-kernel stage of a profiled run:
    algorithmic bytes per launch / event-measured time per launch."""
    hbm_peak, _, src = peaks()
    # single-kernel HBM stages (route / sort / owner_dedup are multi-kernel
    # sequences on the aux stream, reported in `stages` only)
    hbm_stages = ["gather", "refresh", "send_gather", "pool", "segsum", "update"]
    dom = max((n for n in hbm_stages if st[n]["records"]), key=lambda n: st[n]["ms"])
    ds = st[dom]
    achieved = ds["bytes"] / (ds["ms"] * 1e6)
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(f"{key_prefix}/{dom}")
    return {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
            "frac": achieved / hbm_peak, "traffic": traffic, "peak_source": src,
            "bytes_per_launch": ds["bytes"] / ds["records"], "ms_per_launch": ds["ms"] / ds["records"]}


# ----------------------------------------------------------------------------- clocks
class Clocks:
    """nvidia-smi samples (every 50 ms) of SM clocks and throttle reasons.  The
    sampler starts before the warm-up; the timed region is marked with host
    wall-clock times and only the samples inside it are used (the nearest one
    when the region is shorter than the sampling period)."""
    FIELDS = "timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active," \
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_gpu{gpu_index}.csv")
        self.t0 = self.t1 = None

    def start(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "50", "-i", str(self.gpu)], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    @staticmethod
    def _ts(x):
        import datetime
        try:
            return datetime.datetime.strptime(x, "%Y/%m/%d %H:%M:%S.%f").timestamp()
        except ValueError:
            return None

    def stop(self):
        if not self.proc:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        rows = []
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 10:
                continue
            try:
                smv, mxv = float(parts[2]), float(parts[3])
            except ValueError:
                continue
            rs = {n for n, v in zip(names, parts[6:10]) if v.lower().startswith("active")}
            rows.append((self._ts(parts[0]), smv, mxv, rs))
        if not rows:
            return None
        sel = rows
        if self.t0 is not None and self.t1 is not None and all(r[0] is not None for r in rows):
            inside = [r for r in rows if self.t0 <= r[0] <= self.t1]
            mid = 0.5 * (self.t0 + self.t1)
            sel = inside or [min(rows, key=lambda r: abs(r[0] - mid))]
        reasons = set().union(*(r[3] for r in sel))
        return {"sm_mhz": statistics.median(r[1] for r in sel), "sm_max_mhz": max(r[2] for r in sel),
                "samples": len(sel), "samples_in_timed_region": len([r for r in sel if self.t0 is not None
                                                                     and r[0] is not None
                                                                     and self.t0 <= r[0] <= self.t1]),
                "reasons": sorted(reasons)}


# ----------------------------------------------------------------------------- workload
def rank_batches(cfg, seed, rank, P, args=None):
    if args is not None and args.reuse > 0:
        return WL.gen_overlap_batches(cfg, seed, P, rank, args.reuse)
    if args is not None and args.correlated:
        g, rho = args.correlated.split(",")
        return [WL.gen_correlated_batch(cfg, seed, t, rank, groups=int(g), rho=float(rho)) for t in range(P)]
    return [WL.gen_batch(cfg, seed, t, rank) for t in range(P)]


# ----------------------------------------------------------------------------- oracle arms
def oracle_sample_step(cfg, seed, rank, samples, step=0):
    """One oracle step (source routing + Eq. 1/2 step) on a bounded sample."""
    from oracle import routing as OR
    from oracle import step as OS
    keys, offs = WL.gen_batch(cfg, seed, step, rank, batch=samples)
    dout = WL.gen_dout(seed, step, rank, samples * cfg.num_features, cfg.dim, "realistic")
    # the table rows exist before the step (PRF initialisation is table
    # creation, not step work): materialise them outside the timed region
    tab = OS.LazyTable(seed, cfg.dim)
    tab.get(np.unique(keys))
    t0 = time.perf_counter()
    OR.route_source(keys, 1)
    OS.sync_step(tab, [(keys, offs)], [dout], 1e-3, pooling=cfg.pooling)
    return time.perf_counter() - t0


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def tiny_oracle_baseline(seed, steps=10):
    """SURVEY §8(d) oracle timing on the tiny config: 10 synchronous steps of
    the global batch (W = 2 shards x 32 samples), routing + Eq. 1/2 step."""
    from oracle import routing as OR
    from oracle import step as OS
    cfg = WL.CONFIGS["tiny"]
    W = 2
    tab = OS.LazyTable(seed, cfg.dim)
    t0 = time.perf_counter()
    for t in range(steps):
        batches = [WL.gen_batch(cfg, seed, t, r) for r in range(W)]
        douts = [WL.gen_dout(seed, t, r, cfg.batch_local * cfg.num_features, cfg.dim, "realistic") for r in range(W)]
        OR.route_all(batches, W)
        OS.sync_step(tab, batches, douts, 1e-3)
    dt = time.perf_counter() - t0
    return {"value": steps * W * cfg.batch_local / dt, "unit": UNIT, "steps": steps,
            "sample": f"tiny config, {steps} steps of the global batch ({W} x {cfg.batch_local} samples), "
                      f"oracle route_all + sync_step, {dt:.3f} s"}


def cpu_baseline(cfg, seed, min_s=10.0):
    """The oracle on a bounded sample: grow the sample x4 until one step costs
    >= min_s of CPU time (10-30 s) or covers the whole local batch."""
    samples = 1024
    dt = oracle_sample_step(cfg, seed, 0, samples)
    while dt < min_s and samples < cfg.batch_local:
        samples = min(cfg.batch_local, samples * 4)
        dt = oracle_sample_step(cfg, seed, 0, samples)
    return {"value": samples / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "host_cpus": len(os.sched_getaffinity(0)), "cpu_model": cpu_model(),
            "sample": f"{samples} of {cfg.batch_local} samples of one rank's {cfg.name} batch; "
                      f"oracle route_source + sync_step (numpy fp64, single thread), {dt:.2f} s",
            "tiny_10_steps": tiny_oracle_baseline(seed)}


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    # ~1.4 s of oracle work per step: the driver's --steps K --warmup W run
    # stays within a few minutes
    samples = 2048
    for t in range(args.warmup):
        oracle_sample_step(cfg, args.seed, 0, samples, t)
    tot = 0.0
    for t in range(args.steps):
        tot += oracle_sample_step(cfg, args.seed, 0, samples, args.warmup + t)
    v = samples * args.steps / tot
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_json(args, cfg, world),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"{samples} samples per step of one rank's {cfg.name} batch "
                                       "(oracle route_source + sync_step, numpy fp64, 1 thread; table rows "
                                       "materialised before the timer)", "cpu_model": cpu_model()},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_json(args, cfg, world):
    return {"workload": cfg.name, "tables": cfg.num_tables, "total_rows": int(sum(cfg.table_rows)),
            "dim": cfg.dim, "batch_per_gpu": cfg.batch_local, "global_batch": cfg.batch_local * world,
            "bag_len": f"U{{{cfg.bag_len[0]}..{cfg.bag_len[1]}}}", "zipf": cfg.zipf, "pooling": cfg.pooling,
            "micro_batches": args.micro_batches, "schedule": args.schedule, "optimizer": args.optimizer,
            "variant": "E+T (embedding + stand-in tower)" if args.variant == "et" else "E (embedding only)",
            "tower": f"{cfg.tower_layers}x{cfg.tower_hidden} bf16 cuBLAS" if args.variant == "et" else None,
            "dout": "stand-in tower input gradient" if args.variant == "et" else
                    "fixed seeded loss gradient of the pooled rows (N(0, 1e-2))",
            "parallelism": f"tables row-sharded over {world} GPU(s), data-parallel samples",
            "l2": "inputs larger than L2 (tables 4*rows*dim bytes, GB-scale per-step traffic)",
            "pipelined": "DBP (route t+1 on the aux stream)" + (
                f" + FWP ({args.micro_batches} micro-batches, comm/compute streams)" if args.micro_batches > 1
                else "; FWP off (1 micro-batch; FWP at N=2 measured alongside when W > 1)"),
            "exchanges": None if world == 1 else (
                f"rows: {os.environ.get('NEST_A2A', 'fused')} (fused = SM peer stores into IPC-mapped windows), "
                f"counts/keys: {os.environ.get('NEST_ROUTE_XCHG', 'window')}, early push: "
                f"{os.environ.get('NEST_EARLY_PUSH', 'sm')}, direct write-back: "
                f"{'off' if os.environ.get('NEST_DIRECT_WB') == '0' else 'on'}"),
            "tower_trained": bool(getattr(args, "tower_train", False)),
            "tables_in": "HBM" if getattr(args, "tables", "hbm") == "hbm" else
                         "pinned host DRAM (retrieval / refresh / write-back over PCIe)"}


# ----------------------------------------------------------------------------- our arm
def main():
    args = parse()
    cfg = WL.CONFIGS[args.config]
    if args.zipf > 0:
        cfg = cfg.with_(zipf=args.zipf)
    if args.tower_layers > 0:
        cfg = cfg.with_(tower_layers=args.tower_layers)
    if cfg.pooling == "none":
        args.variant = "e"     # the stand-in tower is defined on pooled rows only
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and "RANK" in os.environ:
        pass  # torchrun decides
    if args.micro_batches <= 0:
        # measured best at W = 1, 2, 4 on B200: hiding the
        # All2All behind the tower costs as much compute as it hides, so the
        # default runs one micro-batch and reports N = 2 alongside
        args.micro_batches = 1
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return
    if args.warmup < 3:
        args.warmup = 3
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    from paper_2604_06956_b200 import NestContext, unique_ids
    from paper_2604_06956_b200.runner import Runner

    N = args.micro_batches
    B, F, d = cfg.batch_local, cfg.num_features, cfg.dim
    batches = rank_batches(cfg, args.seed, rank, args.batches, args)
    # --seeds n: the other seeds' batches too (capacities cover all of them)
    extra = [rank_batches(cfg, args.seed + i, rank, args.batches, args) for i in range(1, max(1, args.seeds))]
    K = max(len(k) for k, _ in batches + [b for bs in extra for b in bs])
    # capacities from the actual batches: unique keys per batch bound the
    # received keys per owner (balanced by the row mod W rule) and the rows
    # exchanged per micro-batch (sum_i U_{s,i} <= min(K, N * U_s))
    U = max(len(np.unique(k)) for k, _ in batches + [b for bs in extra for b in bs])
    if world > 1:
        # one configuration on every rank (the exchange windows and the
        # capacity decisions of the count exchange must agree)
        import torch.distributed as dist_
        t = torch.tensor([U, K], device=dev)
        dist_.all_reduce(t, op=dist_.ReduceOp.MAX)
        U, K = int(t[0].item()), int(t[1].item())
    Nctx = max(N, 2) if world > 1 else N      # room for the FWP comparison run
    with_tower = cfg.pooling == "sum" and (args.variant == "et" or not args.no_fwp_compare)
    mb_rows = min(K, Nctx * U) + 1024
    uids = None
    if world > 1:
        obj = [unique_ids() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uids = obj[0]
    ctx = NestContext(cfg.table_rows, d, num_features=F, world=world, rank=rank, pooling=cfg.pooling,
                      max_keys=K + 1024,
                      max_batch=B, max_micro_batches=Nctx, seed=args.seed + 1, init_mode="uniform",
                      tower_layers=cfg.tower_layers if with_tower else 0,
                      tower_hidden=cfg.tower_hidden, nccl_uids=uids, device=dev, optimizer=args.optimizer,
                      max_recv_keys=int(1.5 * U) + 1024 if world > 1 else U + 1024,
                      max_mb_rows=mb_rows,
                      max_owner_mb_rows=int(1.5 * mb_rows) if world > 1 else 0,
                      table_location=args.tables, tower_train=args.tower_train and with_tower, tower_lr=1e-4)
    torch.cuda.synchronize()
    # inputs resident in HBM (value) and pinned host copies (e2e)
    dev_b = [(torch.from_numpy(k).to(dev), torch.from_numpy(o).to(dev), B) for k, o in batches]
    host_b = [(torch.from_numpy(k).pin_memory(), torch.from_numpy(o).pin_memory()) for k, o in batches]
    lr = 1e-3 / (B * world)
    # row-wise AdaGrad: g = G / |B_global|, step size 0.01
    adagrad = (1.0 / (B * world), 0.01) if args.optimizer == "rowwise_adagrad" else None

    def pooled_dtype(variant):
        # the bf16 tower takes bf16 pooled rows straight from the pool kernel
        # (same values as casting the fp32 rows; NEST_BENCH_POOLED_BF16=0: fp32
        # rows + the tower's cast)
        if variant == "et" and os.environ.get("NEST_BENCH_POOLED_BF16", "1") != "0":
            return torch.bfloat16
        return torch.float32

    def make_dout_fn(variant, n_mb):
        if variant == "et":
            douts = {}

            def fn(t, i, pooled):
                key = (i, pooled.shape[0])
                if key not in douts:
                    douts[key] = torch.empty(pooled.shape, dtype=torch.float32, device=dev)
                ctx.tower_fwd_bwd(pooled, douts[key], stream=torch.cuda.current_stream())  # dense lane
                if i == n_mb - 1:
                    # trained tower: one dense AllReduce + SGD per batch (no-op when fixed)
                    ctx.tower_step(stream=torch.cuda.current_stream())
                return douts[key]
            return fn
        fixed = {}

        def fn(t, i, pooled):
            key = (i, pooled.shape[0])
            if key not in fixed:
                g = torch.Generator(device=dev).manual_seed(1000 + i)
                fixed[key] = torch.randn(pooled.shape, generator=g, device=dev) * 1e-2
            return fixed[key]
        return fn

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize()

    def timed(runner, steps, t0, source=None, profile=False, variant=None, dev_b=dev_b):
        """Runs `steps` steps; returns device ms (max over ranks)."""
        dout_fn = make_dout_fn(variant or args.variant, runner.N)
        barrier()
        if profile:
            ctx.profile_enable(True)
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        start.record(runner.compute)
        h2d = d2h = 0
        pending = None   # e2e: (event, pinned row) of the previous step's result read
        if source == "host":
            d2h_stream = torch.cuda.Stream(device=dev)
            res_bufs = [torch.empty((ctx.dim,), dtype=runner.pooled_dtype, pin_memory=True) for _ in range(2)]
        for s in range(steps):
            t = t0 + s
            cur, nxt = t % len(dev_b), (t + 1) % len(dev_b)
            if source == "host":
                # e2e: this step's NEXT batch arrives from pinned host memory
                hk, ho = host_b[nxt]
                nk = torch.empty(hk.shape, dtype=hk.dtype, device=dev)
                no = torch.empty(ho.shape, dtype=ho.dtype, device=dev)
                nk.copy_(hk, non_blocking=True)
                no.copy_(ho, non_blocking=True)
                h2d += hk.numel() * 8 + ho.numel() * 4
                nb = (nk, no, B)
            else:
                nb = dev_b[nxt]
            # the current batch was routed by the previous step (DBP); only an
            # unprimed runner routes it here
            outs = runner.step(dev_b[cur], nb, dout_fn, keep_outputs=True)
            if source == "host":
                # the step's result (a pooled row) read back to the host, ordered
                # after the step's work on the embedding lane; the host waits for
                # step t-1's read after step t is enqueued (one step of lag keeps
                # the queue full)
                if pending is not None:
                    pending[0].synchronize()
                    float(pending[1][0])
                row = outs[-1][0]
                buf = res_bufs[s % 2]
                d2h_stream.wait_stream(runner.compute)
                with torch.cuda.stream(d2h_stream):
                    buf.copy_(row, non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(d2h_stream)
                outs[-1].record_stream(d2h_stream)
                pending = (ev, buf)
                d2h += row.numel() * row.element_size()
        if pending is not None:
            runner.compute.wait_stream(d2h_stream)   # the last result read is inside the timed region
        end.record(runner.join())
        torch.cuda.synchronize()
        if pending is not None:
            float(pending[1][0])
        ms = start.elapsed_time(end)
        prof = None
        if profile:
            ctx.profile_enable(False)
            prof = ctx.profile_read()
            if args.trace:
                prof["records"] = ctx.profile_records()
        if world > 1:
            tt = torch.tensor([ms], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = float(tt.item())
        return ms, prof, h2d, d2h

    sched_cache = {}
    # the route's host sync after the tower is queued (E+T) / after the
    # backward is queued (E): DESIGN.md §1, Runner(route_end=...)
    rend = {"et": "before_grad", "e": "after_grad"}
    runner = Runner(ctx, N=N, schedule=args.schedule, pipelined=True, lr_over_B=lr, adagrad=adagrad,
                    sched_cache=sched_cache, route_end=rend[args.variant],
                    pooled_dtype=pooled_dtype(args.variant))
    clocks = Clocks(local)
    clocks.start()   # before the warm-up: nvidia-smi's first sample takes ~0.1-0.3 s
    timed(runner, args.warmup, 0)
    clocks.mark_start()
    ms, prof, _, _ = timed(runner, args.steps, args.warmup, profile=True)
    clocks.mark_end()
    clk = clocks.stop()
    trace_records = prof.get("records")
    value = B * world * args.steps / (ms / 1e3)
    # FWP payload of the last routed batch: sum_i |K(M_i)| vs |K(B)|
    info = ctx.slot_info(runner.t % 2)
    cluster_ms = None
    if N > 1 and args.schedule.startswith("clustered"):
        # the GPU greedy on one batch, alone (its cost per batch; inside the
        # step for "clustered", outside for "clustered-offline")
        kk, oo, _ = dev_b[0]
        ctx.fwp_schedule(kk, oo, B, N, "clustered")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            ctx.fwp_schedule(kk, oo, B, N, "clustered")
        e1.record()
        torch.cuda.synchronize()
        cluster_ms = e0.elapsed_time(e1) / 3
    fwp_stats = {"N": N, "schedule": args.schedule, "cluster_ms_per_batch": cluster_ms,
                 "uniq_keys": int(info.uniq),
                 "sum_mb_uniq": int(sum(info.mb_uniq[i] for i in range(N))),
                 "alpha": (sum(info.mb_uniq[i] for i in range(N)) / info.uniq) if info.uniq else None}

    seed_ms, seed_median_ms = None, None
    if extra:
        # the same timed loop on every seed's batches, median
        # reported (the profiled statistics stay those of the first seed)
        seed_ms = [ms / args.steps]
        for i, bs in enumerate(extra):
            db = [(torch.from_numpy(k).to(dev), torch.from_numpy(o).to(dev), B) for k, o in bs]
            rs = Runner(ctx, N=N, schedule=args.schedule, pipelined=True, lr_over_B=lr, adagrad=adagrad,
                        sched_cache={}, route_end=rend[args.variant], pooled_dtype=pooled_dtype(args.variant))
            rs.t = runner.t + 16 * (i + 1)
            timed(rs, args.warmup, rs.t, dev_b=db)
            ms_i, _, _, _ = timed(rs, args.steps, rs.t, dev_b=db)
            seed_ms.append(ms_i / args.steps)
            rs._hold, rs.outs = [], []
            runner.t = rs.t          # later runners continue from the last routed slot
            del db
        seed_median_ms = statistics.median(seed_ms)
    if seed_median_ms is not None:
        ms = seed_median_ms * args.steps
        value = B * world * args.steps / (ms / 1e3)
    # e2e through the public API with host inputs (copies inside the timed region)
    e2e = None
    # release the timed runner's held outputs (gen-rec: 17 GB per step) before
    # the other runners allocate theirs
    runner._hold, runner.outs = [], []
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    if not args.no_e2e:
        # e2e: fresh device copies every step -- an offline partition is keyed
        # by the device batch, so this run clusters inside the step (conservative)
        r2 = Runner(ctx, N=N, schedule="clustered" if args.schedule == "clustered-offline" else args.schedule,
                    pipelined=True, lr_over_B=lr, adagrad=adagrad, route_end=rend[args.variant],
                    pooled_dtype=pooled_dtype(args.variant))
        r2.t = runner.t
        timed(r2, 2, runner.t, source="host")
        ms_e, _, h2d, d2h = timed(r2, args.steps, r2.t, source="host")
        counts_bytes = 4 * (world * world * (N + 2) + N + 1)
        e2e = {"value": B * world * args.steps / (ms_e / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": h2d // args.steps,
               "d2h_bytes_per_step": d2h // args.steps + counts_bytes,
               "ms_per_step": ms_e / args.steps}

    # the same step with the stand-in dense tower (FWP's overlap partner):
    # N = 1 (no FWP) and, when there is an All2All to hide, N = 2 (FWP)
    def tower_run(Nv, t0):
        r1 = Runner(ctx, N=Nv, schedule=args.schedule if Nv > 1 else "sequential", pipelined=True,
                    sched_cache=sched_cache, route_end=rend["et"],
                    lr_over_B=lr, adagrad=adagrad, pooled_dtype=pooled_dtype("et"))
        r1.t = t0
        timed(r1, 3, r1.t, variant="et")
        k2 = max(5, args.steps // 2)
        ms1, prof1, _, _ = timed(r1, k2, r1.t, profile=True, variant="et")
        sm, st1 = prof1["summary"], prof1["stages"]
        tw = st1["tower"]
        out = {"N": Nv, "steps": k2, "ms_per_step": ms1 / k2, "samples_per_s": B * world * k2 / (ms1 / 1e3),
               "roofline": roofline_from(st1, f"{cfg.name}/W{world}/N{Nv}"),
               "tower_ms_per_step": tw["ms"] / k2,
               "tower_tflops": (tw["bytes"] + st1["tower_dw"]["bytes"]) / ((tw["ms"] + st1["tower_dw"]["ms"]) * 1e9)
               if tw["ms"] else None}
        if world > 1:
            out["a2a_ms_per_step"] = sm["a2a_ms"] / k2
            out["a2a_exposed_ms_per_step"] = sm["a2a_exposed_ms"] / k2
            out["a2a_exposed_ratio"] = sm["a2a_exposed_ms"] / sm["a2a_ms"] if sm["a2a_ms"] else None
        return out, r1.t

    def embedding_run(Nv, t0):
        r1 = Runner(ctx, N=Nv, schedule=args.schedule, pipelined=True, lr_over_B=lr, adagrad=adagrad,
                    sched_cache=sched_cache, route_end=rend["e"],
                    pooled_dtype=pooled_dtype("e"))
        r1.t = t0
        timed(r1, 3, r1.t, variant="e")
        ms1, prof1, _, _ = timed(r1, args.steps, r1.t, profile=True, variant="e")
        st1 = prof1["stages"]
        return {"N": Nv, "steps": args.steps, "ms_per_step": ms1 / args.steps,
                "samples_per_s": B * world * args.steps / (ms1 / 1e3),
                # the same roofline kernel without the tower's GEMMs beside it
                "roofline": roofline_from(st1, f"{cfg.name}/W{world}/N{Nv}"),
                "whole_step_hbm": whole_step_hbm(st1, args.steps, ms1 / args.steps),
                "stage_ms_per_step": {k: v["ms"] / args.steps for k, v in st1.items() if v["records"]}}, r1.t

    # host-DRAM tier (NEXT-3): the retrieval's PCIe rate against the measured
    # pinned H2D copy, and the step with DBP off (route + retrieval inline)
    host_tier = None
    if args.tables == "host":
        hsrc = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
        ddst = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
        ddst.copy_(hsrc, non_blocking=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(4):
            ddst.copy_(hsrc, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        h2d_peak = 4 * (1 << 30) / (e0.elapsed_time(e1) / 1e3) / 1e9
        del hsrc, ddst
        row = d * 4
        g = prof["stages"]["gather"]
        rname_h = "emb_repush" if prof["stages"]["emb_repush"]["records"] else "refresh"
        rf = prof["stages"][rname_h]
        seq = Runner(ctx, N=N, schedule=args.schedule, pipelined=False, lr_over_B=lr, adagrad=adagrad,
                     pooled_dtype=pooled_dtype(args.variant))
        seq.t = runner.t + 4
        timed(seq, 2, seq.t)
        ms_seq, _, _, _ = timed(seq, max(5, args.steps // 2), seq.t)
        host_tier = {"pcie_h2d_copy_gbs": h2d_peak,
                     "retrieval_gbs": g["units"] * row / (g["ms"] * 1e6) if g["ms"] else None,
                     "retrieval_frac_of_h2d_copy": (g["units"] * row / (g["ms"] * 1e6)) / h2d_peak if g["ms"] else None,
                     "retrieval_ms_per_step": g["ms"] / args.steps,
                     "refresh_ms_per_step": rf["ms"] / args.steps,
                     "pcie_h2d_bytes_per_step": (g["units"] + rf["units"]) * row / args.steps,
                     "pcie_d2h_bytes_per_step": g["units"] * row / args.steps,
                     "ms_per_step_dbp": ms / args.steps,
                     "ms_per_step_sequential": ms_seq / max(5, args.steps // 2)}

    with_tower_runs, embedding_only, zero_copy = None, None, None
    if not args.no_fwp_compare:
        tnext = runner.t + args.steps + 8
        if args.variant == "et":
            with_tower_runs = {f"N{N}": {"N": N, "ms_per_step": ms / args.steps, "samples_per_s": value,
                                         "a2a_ms_per_step": prof["summary"]["a2a_ms"] / args.steps,
                                         "a2a_exposed_ms_per_step": prof["summary"]["a2a_exposed_ms"] / args.steps,
                                         "main_run": True}}
            if world > 1:
                N2 = 2 if N == 1 else 1
                if N2 <= ctx.cfg.max_micro_batches:
                    res, tnext = tower_run(N2, tnext)
                    with_tower_runs[f"N{N2}"] = res
            embedding_only, tnext = embedding_run(N, tnext + 8)
            if N == 1 and args.tables == "hbm" and cfg.pooling == "sum" and \
                    (world == 1 or os.environ.get("NEST_A2A", "fused") == "fused"):
                # zero-copy retrieval: the same steps without the
                # DBP retrieval copy and refresh -- the shard read in place
                ctx.set_zero_copy(True)
                zc_et, tnext = tower_run(1, tnext + 8)
                zc_e, tnext = embedding_run(1, tnext + 8)
                ctx.set_zero_copy(False)
                zero_copy = {"note": "HBM tables: no retrieval copy (R4); W=1: no refresh (R5), pool and fused "
                                     "update read the shard in place; W>1: owners push and update their shard "
                                     "rows in place (re-push kept); same results (parity tests)",
                             "et": {k: zc_et[k] for k in ("ms_per_step", "samples_per_s", "roofline")},
                             "e": {k: zc_e[k] for k in ("ms_per_step", "samples_per_s", "roofline",
                                                        "whole_step_hbm")}}
        elif with_tower:
            with_tower_runs = {}
            for Nv in ([1, 2] if world > 1 and ctx.cfg.max_micro_batches >= 2 else [1]):
                res, tnext = tower_run(Nv, tnext)
                with_tower_runs[f"N{Nv}"] = res

    if rank == 0:
        hbm_peak, bf16_peak, src = peaks()
        st = prof["stages"]
        steps = args.steps
        stages = {}
        for name, s in st.items():
            if s["records"] == 0:
                continue
            e = {"ms_per_step": s["ms"] / steps, "launches_per_step": s["launches"] / steps,
                 "records_per_step": s["records"] / steps}
            if name in ("tower", "tower_dw"):
                e["tflops"] = s["bytes"] / (s["ms"] * 1e9) if s["ms"] else None
            elif name in ("emb_a2a", "grad_a2a", "key_a2a"):
                e["nvlink_gbs"] = s["bytes"] / (s["ms"] * 1e6) if s["ms"] else None
            else:
                gbs = s["bytes"] / (s["ms"] * 1e6) if s["ms"] else None
                e["hbm_gbs"] = gbs
                e["frac_of_measured_hbm"] = gbs / hbm_peak if gbs else None
            stages[name] = e
        roofline = roofline_from(st, f"{cfg.name}/W{world}/N{N}")
        summ = prof["summary"]
        a2a = None
        if world > 1:
            a2a_bytes = st["emb_a2a"]["bytes"] + st["grad_a2a"]["bytes"]
            a2a_ms = summ["a2a_ms"]
            a2a = {"physical_ms_per_step": a2a_ms / steps,
                   "exposed_ms_per_step": summ["a2a_exposed_ms"] / steps,
                   "exposed_ratio": summ["a2a_exposed_ms"] / a2a_ms if a2a_ms else None,
                   "nvlink_gbs_per_gpu": a2a_bytes / (a2a_ms * 1e6) if a2a_ms else None,
                   "frac_of_peer_770": (a2a_bytes / (a2a_ms * 1e6)) / NVLINK_PEER_GBS if a2a_ms else None,
                   "frac_of_nominal_900": (a2a_bytes / (a2a_ms * 1e6)) / NVLINK_NOMINAL_GBS if a2a_ms else None,
                   # all-to-all ceiling measured by scripts/p2p_probe.cu (SM remote
                   # stores, every GPU exchanging with every other): 691 GB/s at
                   # 2 GPUs, 403 GB/s at 4 GPUs per GPU per direction
                   "probe_all2all_ceiling_gbs": {2: 691.2, 4: 403.3}.get(world),
                   "transport": os.environ.get("NEST_A2A", "fused"),
                   "with_tower": with_tower_runs}
        # the dual-buffer refresh (fused with the re-push under the early push)
        rname = "emb_repush" if st["emb_repush"]["records"] else "refresh"
        rs = st[rname]
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline(cfg, args.seed)
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": config_json(args, cfg, world), "roofline": roofline,
                "whole_step_hbm": whole_step_hbm(st, steps, ms / steps), "cpu_baseline": cpu,
                "e2e": e2e, "gpu_launches": int(summ["launches"]), "clocks": clk, "a2a": a2a,
                "stages": stages,
                "trace": {"span_ms_per_step": summ["span_ms"] / steps,
                          "compute_busy_ms_per_step": summ["compute_busy_ms"] / steps},
                "dbp": {"refresh_ms_per_step": rs["ms"] / max(1, rs["records"]),
                        "refresh_stage": rname,
                        "refreshed_rows_per_step": rs["units"] / max(1, rs["records"]),
                        # the prefetch gather copies U_o - I rows (the pending update's keys
                        # are skipped and supplied by the refresh), so U_o = gathered + I
                        "gathered_rows_per_step": st["gather"]["units"] / max(1, st["gather"]["records"]),
                        "owner_unique_per_step": (st["gather"]["units"] + rs["units"]) / max(1, st["gather"]["records"]),
                        "intersection_ratio": (rs["units"] / (st["gather"]["units"] + rs["units"])
                                               if st["gather"]["units"] + rs["units"] else None)},
                "fwp": dict(fwp_stats, with_tower=with_tower_runs),
                "seeds": None if seed_ms is None else {"first": args.seed, "n": len(seed_ms),
                                                       "ms_per_step": seed_ms, "value_is": "median"},
                "embedding_only": embedding_only, "zero_copy": zero_copy}
        if host_tier is not None:
            line["host_tier"] = host_tier
        if args.trace:
            json.dump({"stages": st, "summary": summ, "records": trace_records}, open(args.trace, "w"), indent=1)
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.barrier(device_ids=[local])
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
