"""Step orchestration over the C ABI: the DBP + FWP call order.

Only sequencing lives here (which nest_* call, on which stream, in which
order); all work runs in libnest.so.  The order follows the paper:

* DBP: Key Routing + Retrieval of batch t+1 (``nest_route`` on the
  aux stream) overlaps the window of batch t; after update(t) the dual-buffer
  refresh copies the intersection Active -> Prefetch; the slot roles swap.
* FWP: the window of batch t runs N micro-batches; the
  embedding All2All of micro-batch i+1 is issued on the comm stream before
  micro-batch i's dense compute ("communication launched as early as
  possible"), gradients of micro-batch i follow its compute, and the single
  deferred update runs after micro-batch N.
"""
from __future__ import annotations

from typing import Callable, List, Optional

import torch

from . import NestContext


class Runner:
    """Drives one rank through steps.  `dout_fn(t, i, pooled_i) -> dout_i`
    supplies the loss gradient of micro-batch i (LIN: a fixed tensor, QUAD:
    pooled itself, tower: the stand-in tower's input gradient)."""

    def __init__(self, ctx: NestContext, N: int = 1, schedule: str = "sequential",
                 pipelined: bool = True, lr_over_B: float = 2.0 ** -10):
        self.ctx, self.N, self.schedule, self.pipelined = ctx, N, schedule, pipelined
        self.lr = lr_over_B
        dev = ctx.device
        self.compute = torch.cuda.Stream(device=dev)
        # comm stream at high priority: its CTAs are scheduled first as SMs free up
        self.comm = torch.cuda.Stream(device=dev, priority=-1) if ctx.world > 1 else self.compute
        self.aux = torch.cuda.Stream(device=dev)
        self.t = 0
        self.primed = False
        self.outs: List[torch.Tensor] = []
        self.sched = {}

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
        with torch.cuda.stream(self.compute):   # allocation stream = use stream
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
        cs, ms = self.compute, self.comm
        cs.wait_stream(torch.cuda.current_stream(ctx.device))   # batch uploads
        if not self.pipelined or not self.primed:
            self._route(a, keys, offs, B, cs)
            self.primed = True
        outs = self.out_buffers(a)
        self.outs = outs if keep_outputs else []
        # comm stream: emb_1, emb_2, grad_1, emb_3, grad_2, ... (emb A2A of
        # micro-batch i+1 queued before grad A2A of i); compute stream:
        # pool_i, tower_i, segsum_i -- compute never waits for a later
        # micro-batch's communication
        ctx.lookup_prefetch(a, 0, cs, ms)
        for i in range(self.N):
            ctx.lookup_fwd(a, i, outs[i], cs, ms)
            if i + 1 < self.N:
                ctx.lookup_prefetch(a, i + 1, cs, ms)
            with torch.cuda.stream(cs):
                dout = dout_fn(self.t, i, outs[i]) if dout_fn else outs[i]
            if i == self.N - 1 and self.pipelined and next_batch is not None:
                nk, no, nB = next_batch
                self.aux.wait_stream(torch.cuda.current_stream(ctx.device))
                self._route(p, nk, no, nB, self.aux)      # host blocks for counts here
            ctx.grad_bwd_update(a, i, dout, self.lr, cs, ms)
        if self.pipelined and next_batch is not None:
            ctx.dbp_refresh(a, p, cs)
        self.t += 1
        return outs
