"""Step orchestration over the C ABI: the DBP + FWP call order.

Only sequencing lives here (which nest_* call, on which stream, in which
order); all work runs in libnest.so.  The order follows the paper:

* DBP: Key Routing + Retrieval of batch t+1 (``nest_route`` on the
  aux stream) overlaps the window of batch t; after update(t) the dual-buffer
  refresh overwrites the intersection in the prefetch slot; the slots swap.
* FWP: the window of batch t runs N micro-batches on
  separate lanes -- a comm stream (owner send gather + All2All, issued as
  early as possible), an embedding stream (pool / segment-sum, the
  sparse side of forward / backward) and a dense stream (the stand-in tower).
  Pooling micro-batch i+1 and the gradients of micro-batch i run while the
  tower computes; the single deferred update follows micro-batch N.
"""
from __future__ import annotations

import os
from typing import Callable, List, Optional

import torch

from . import NestContext


_GREEN = {}


def _green_streams(dev, nsm: int, sparse_prios, dense_prios):
    """Streams on two green contexts splitting the device's SMs: `nsm` SMs for
    the sparse lanes, the remainder for the dense lane (CUDA >= 12.4)."""
    from cuda.bindings import driver as cu

    def ok(r):
        err, *vals = r
        if err != cu.CUresult.CUDA_SUCCESS:
            raise RuntimeError(f"green context setup failed: {err}")
        return vals[0] if len(vals) == 1 else tuple(vals)

    key = (dev.index, nsm)
    if key not in _GREEN:
        torch.cuda.init()
        cudev = ok(cu.cuDeviceGet(dev.index))
        res = ok(cu.cuDeviceGetDevResource(cudev, cu.CUdevResourceType.CU_DEV_RESOURCE_TYPE_SM))
        groups, _n, rem = ok(cu.cuDevSmResourceSplitByCount(1, res, 0, nsm))
        ctxs = []
        for r in (groups[0], rem):
            desc = ok(cu.cuDevResourceGenerateDesc([r], 1))
            ctxs.append(ok(cu.cuGreenCtxCreate(desc, cudev, cu.CUgreenCtxCreate_flags.CU_GREEN_CTX_DEFAULT_STREAM)))
        _GREEN[key] = ctxs
    sparse_ctx, dense_ctx = _GREEN[key]

    def mk(gctx, prio):
        s = ok(cu.cuGreenCtxStreamCreate(gctx, cu.CUstream_flags.CU_STREAM_NON_BLOCKING.value, prio))
        return torch.cuda.ExternalStream(int(s), device=dev)
    return [mk(sparse_ctx, p) for p in sparse_prios], [mk(dense_ctx, p) for p in dense_prios]


class Runner:
    """Drives one rank through steps.  `dout_fn(t, i, pooled_i) -> dout_i`
    supplies the loss gradient of micro-batch i on the dense stream (LIN: a
    fixed tensor, QUAD: pooled itself, tower: the stand-in tower's input
    gradient)."""

    def __init__(self, ctx: NestContext, N: int = 1, schedule: str = "sequential",
                 pipelined: bool = True, lr_over_B: float = 2.0 ** -10, pooled_dtype=None,
                 adagrad=None, sched_cache: Optional[dict] = None, route_end: Optional[str] = None):
        # schedule: "sequential", "clustered" (the GPU greedy inside every
        # route), or "clustered-offline" (clustering "can be performed
        # asynchronously on CPU or offline": the partition of a batch is
        # computed once, by the same GPU greedy, the first time the batch is
        # seen, and reused -- e.g. precomputed by the data pipeline)
        self.ctx, self.N, self.schedule, self.pipelined = ctx, N, schedule, pipelined
        self.sched_cache = sched_cache if sched_cache is not None else {}
        # when the DBP route of the next batch does its host sync (nest_route_end):
        # "after_grad" (default) once the window's backward is queued, so the
        # compute lane has work while the host waits for the counts; or
        # "before_grad" right after the dense lane's work (the stand-in tower)
        # is queued -- that work covers the wait, and the gather / owner
        # dedup then run beside the tower instead of beside the segment-sum
        # (NEST_ROUTE_END overrides)
        self.route_end_mode = os.environ.get("NEST_ROUTE_END") or route_end or "after_grad"
        self.lr = lr_over_B
        # row-wise AdaGrad contexts: (grad_scale, lr) of nest_grad_bwd_update_adagrad
        self.adagrad = adagrad
        # bf16: pooled rows for a bf16 dense consumer (nest_lookup_fwd_bf16)
        self.pooled_dtype = pooled_dtype or torch.float32
        self._hold: List[torch.Tensor] = []
        dev = ctx.device
        # block-scheduling priorities (lower = scheduled first as SMs free up):
        # dense tower > comm > embedding, so the overlapped sparse work takes
        # the SMs the GEMMs leave (NEST_LANE_PRIORITIES="dense,comm,emb")
        pd, pc, pe = (int(x) for x in os.environ.get("NEST_LANE_PRIORITIES", "-2,-1,0").split(","))
        # 3: dense / embedding / comm lanes; 2: the paper's computation +
        # communication streams (NEST_LANES)
        self.lanes = int(os.environ.get("NEST_LANES", "3"))
        green = int(os.environ.get("NEST_GREEN_SMS", "0"))
        if green > 0:
            # hard SM partition (green contexts): the sparse lanes (embedding,
            # comm, DBP lookahead) get `green` SMs, the dense tower the rest
            sparse_s, dense_s = _green_streams(dev, green, [pe, pc, -5, 0], [pd, 0])
            self.compute, comm, self.aux, sort_s = sparse_s
            self.comm = comm if ctx.world > 1 else self.compute
            self.dense, dw_s = dense_s
            # the library's sort stream with the sparse lanes, the tower's dW
            # stream with the dense lane
            ctx.set_streams(sort_stream=sort_s, tower_dw_stream=dw_s if ctx.cfg.tower_layers > 0 else None)
            self._green_keep = (sort_s, dw_s)
        else:
            self.compute = torch.cuda.Stream(device=dev, priority=pe)            # embedding lane
            self.comm = torch.cuda.Stream(device=dev, priority=pc) if ctx.world > 1 else self.compute
            self.dense = torch.cuda.Stream(device=dev, priority=pd)              # tower lane
            # DBP lookahead (route / owner dedup / gather / early push of batch
            # t+1; its occurrence sort runs on the library's lowest-priority
            # stream): NEST_AUX_PRIORITY, default -5 (the highest), so its many
            # short kernels are not queued behind the window's long-running
            # blocks -- r02 A/B, 2 rounds each: W=1 E step 1.30 vs 1.36-1.52 ms
            # and the E+T segment-sum roofline 0.45-0.49 vs 0.37-0.38 at equal
            # E+T throughput (within noise); W=2 E 2.58-2.63 vs 2.75-2.85 ms
            self.aux = torch.cuda.Stream(device=dev, priority=int(os.environ.get("NEST_AUX_PRIORITY", "-5")))
        self.t = 0
        self.primed = False
        self.outs: List[torch.Tensor] = []
        self.sched = {}
        self._ev_pool = [torch.cuda.Event() for _ in range(8)]
        self._ev_dense = [torch.cuda.Event() for _ in range(8)]

    # -- helpers ---------------------------------------------------------------
    def _grad(self, slot, mb, dout, cs, ms):
        if self.adagrad is not None:
            self.ctx.grad_bwd_update_adagrad(slot, mb, dout, self.adagrad[0], self.adagrad[1], cs, ms)
        else:
            self.ctx.grad_bwd_update(slot, mb, dout, self.lr, cs, ms)

    def _schedule(self, slot, keys, offs, B, stream):
        if self.schedule == "clustered-offline" and self.N > 1:
            key = (keys.data_ptr(), int(keys.numel()), offs.data_ptr(), B, self.N)
            if key not in self.sched_cache:
                self.sched_cache[key] = self.ctx.fwp_schedule(keys, offs, B, self.N, "clustered", stream=stream)
            perm, mbo = self.sched_cache[key]
        else:
            mode = "clustered" if self.schedule.startswith("clustered") else self.schedule
            perm, mbo = self.ctx.fwp_schedule(keys, offs, B, self.N, mode, stream=stream)
        self.sched[slot] = (perm, mbo)
        return perm, mbo

    def _route(self, slot, keys, offs, B, stream):
        perm, mbo = self._schedule(slot, keys, offs, B, stream)
        self.ctx.route(slot, keys, offs, B, perm=perm, mb_offsets=mbo, N=self.N, stream=stream)

    def _route_begin(self, slot, keys, offs, B, stream):
        """DBP route of the next batch, first half (enqueue only): its host
        sync happens in route_end, after the window's backward is enqueued, so
        the compute lane never idles while the host waits for the counts."""
        perm, mbo = self._schedule(slot, keys, offs, B, stream)
        self.ctx.route_begin(slot, keys, offs, B, perm=perm, mb_offsets=mbo, N=self.N, stream=stream)

    def out_buffers(self, slot) -> List[torch.Tensor]:
        info = self.ctx.slot_info(slot)
        outs = []
        with torch.cuda.stream(self.compute):   # allocation stream = producing stream
            for i in range(self.N):
                rows = int(info.mb_out_rows[i])
                outs.append(torch.empty((rows, self.ctx.dim), dtype=self.pooled_dtype,
                                        device=self.ctx.device))
        return outs

    # -- one step ---------------------------------------------------------------
    def step(self, batch, next_batch=None, dout_fn: Optional[Callable] = None,
             keep_outputs: bool = True):
        """Run the window of `batch` (already routed when pipelined) and, when
        pipelined, route `next_batch` into the other slot."""
        ctx = self.ctx
        keys, offs, B = batch
        a, p = self.t % 2, (self.t + 1) % 2
        cs, ms, ds = self.compute, self.comm, self.dense
        cs.wait_stream(torch.cuda.current_stream(ctx.device))   # batch uploads
        if not self.pipelined or not self.primed:
            self._route(a, keys, offs, B, cs)
            self.primed = True
        outs = self.out_buffers(a)
        self.outs = outs if keep_outputs else []
        # a bf16 dense consumer reads the pooled rows in place after this call
        # returns (the tower's deferred dW GEMMs, which alternate two buffer
        # sets): keep them allocated until the step after next has enqueued its
        # tower calls, which wait for those GEMMs (fp32 rows are cast into the
        # tower's own buffer first: nothing to hold)
        keep = 3 if self.pooled_dtype == torch.bfloat16 else 1
        self._hold = (self._hold + [outs])[-keep:]
        if self.lanes == 2:
            return self._step_two_lanes(a, p, outs, next_batch, dout_fn)
        # embedding lane: pool_0, pool_1, seg_0, pool_2, seg_1, ... (pool of
        # micro-batch i+1 is queued before the gradients of i); comm lane:
        # emb_0, emb_1, grad_0, emb_2, grad_1, ...; dense lane: tower_i
        ctx.lookup_prefetch(a, 0, cs, ms)
        ctx.lookup_fwd(a, 0, outs[0], cs, ms)
        self._ev_pool[0].record(cs)
        for i in range(self.N):
            if i + 1 < self.N:
                ctx.lookup_prefetch(a, i + 1, cs, ms)
                ctx.lookup_fwd(a, i + 1, outs[i + 1], cs, ms)
                self._ev_pool[i + 1].record(cs)
            route_next = i == self.N - 1 and self.pipelined and next_batch is not None
            if route_next:
                # DBP: route + retrieval of batch t+1 on the aux lane, inside window t
                nk, no, nB = next_batch
                self.aux.wait_stream(torch.cuda.current_stream(ctx.device))
                self._route_begin(p, nk, no, nB, self.aux)
            ds.wait_event(self._ev_pool[i])
            with torch.cuda.stream(ds):
                dout = dout_fn(self.t, i, outs[i]) if dout_fn else outs[i]
            self._ev_dense[i].record(ds)
            cs.wait_event(self._ev_dense[i])
            if route_next and self.route_end_mode == "before_grad":
                ctx.route_end(p)      # host blocks for the counts; the dense lane is busy
            self._grad(a, i, dout, cs, ms)
            if route_next and self.route_end_mode != "before_grad":
                ctx.route_end(p)      # host blocks for the counts here, the window is queued
        if self.pipelined and next_batch is not None:
            ctx.dbp_refresh(a, p, cs)
        self.t += 1
        return outs

    def _step_two_lanes(self, a, p, outs, next_batch, dout_fn):
        """The paper's two-stream plan: one computation stream runs
        pool_i, tower_i, segsum_i back to back (each on the whole GPU); the
        communication stream runs emb A2A_{i+1} and grad A2A_i as early as
        possible, overlapping the computation of neighbouring micro-batches."""
        ctx = self.ctx
        cs, ms = self.dense, self.comm
        cs.wait_stream(self.compute)          # batch uploads / primed route
        ctx.lookup_prefetch(a, 0, cs, ms)
        ctx.lookup_fwd(a, 0, outs[0], cs, ms)
        for i in range(self.N):
            if i + 1 < self.N:
                ctx.lookup_prefetch(a, i + 1, cs, ms)
            route_next = i == self.N - 1 and self.pipelined and next_batch is not None
            if route_next:
                nk, no, nB = next_batch
                self.aux.wait_stream(torch.cuda.current_stream(ctx.device))
                self._route_begin(p, nk, no, nB, self.aux)
            with torch.cuda.stream(cs):
                dout = dout_fn(self.t, i, outs[i]) if dout_fn else outs[i]
            self._grad(a, i, dout, cs, ms)
            if route_next:
                ctx.route_end(p)
            if i + 1 < self.N:
                ctx.lookup_fwd(a, i + 1, outs[i + 1], cs, ms)
        if self.pipelined and next_batch is not None:
            ctx.dbp_refresh(a, p, cs)
        self.compute.wait_stream(cs)
        self.t += 1
        return outs

    def join(self, stream=None):
        """Make `stream` (default: the embedding lane) wait for every lane."""
        s = stream or self.compute
        for other in (self.comm, self.dense, self.aux):
            if other is not s:
                s.wait_stream(other)
        self.ctx.join(s)
        return s
