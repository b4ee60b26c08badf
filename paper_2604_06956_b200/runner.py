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

from typing import Callable, List, Optional

import torch

from . import NestContext


class Runner:
    """Drives one rank through steps.  `dout_fn(t, i, pooled_i) -> dout_i`
    supplies the loss gradient of micro-batch i on the dense stream (LIN: a
    fixed tensor, QUAD: pooled itself, tower: the stand-in tower's input
    gradient)."""

    def __init__(self, ctx: NestContext, N: int = 1, schedule: str = "sequential",
                 pipelined: bool = True, lr_over_B: float = 2.0 ** -10):
        self.ctx, self.N, self.schedule, self.pipelined = ctx, N, schedule, pipelined
        self.lr = lr_over_B
        dev = ctx.device
        self.compute = torch.cuda.Stream(device=dev)            # embedding lane
        # comm lane at high priority: its kernels are scheduled first as SMs free up
        self.comm = torch.cuda.Stream(device=dev, priority=-1) if ctx.world > 1 else self.compute
        self.dense = torch.cuda.Stream(device=dev)              # tower lane
        self.aux = torch.cuda.Stream(device=dev)                # DBP lookahead
        self.t = 0
        self.primed = False
        self.outs: List[torch.Tensor] = []
        self.sched = {}
        self._ev_pool = [torch.cuda.Event() for _ in range(8)]
        self._ev_dense = [torch.cuda.Event() for _ in range(8)]

    # -- helpers ---------------------------------------------------------------
    def _schedule(self, slot, keys, offs, B, stream):
        perm, mbo = self.ctx.fwp_schedule(keys, offs, B, self.N, self.schedule, stream=stream)
        self.sched[slot] = (perm, mbo)
        return perm, mbo

    def _route(self, slot, keys, offs, B, stream):
        perm, mbo = self._schedule(slot, keys, offs, B, stream)
        self.ctx.route(slot, keys, offs, B, perm=perm, mb_offsets=mbo, N=self.N, stream=stream)

    def out_buffers(self, slot) -> List[torch.Tensor]:
        info = self.ctx.slot_info(slot)
        outs = []
        with torch.cuda.stream(self.compute):   # allocation stream = producing stream
            for i in range(self.N):
                rows = int(info.mb_out_rows[i])
                outs.append(torch.empty((rows, self.ctx.dim), dtype=torch.float32,
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
            ds.wait_event(self._ev_pool[i])
            with torch.cuda.stream(ds):
                dout = dout_fn(self.t, i, outs[i]) if dout_fn else outs[i]
            self._ev_dense[i].record(ds)
            cs.wait_event(self._ev_dense[i])
            if i == self.N - 1 and self.pipelined and next_batch is not None:
                nk, no, nB = next_batch
                self.aux.wait_stream(torch.cuda.current_stream(ctx.device))
                self._route(p, nk, no, nB, self.aux)      # host blocks for counts here
            ctx.grad_bwd_update(a, i, dout, self.lr, cs, ms)
        if self.pipelined and next_batch is not None:
            ctx.dbp_refresh(a, p, cs)
        self.t += 1
        return outs

    def join(self, stream=None):
        """Make `stream` (default: the embedding lane) wait for every lane."""
        s = stream or self.compute
        for other in (self.comm, self.dense, self.aux):
            if other is not s:
                s.wait_stream(other)
        return s
