"""Symbolic NestPipe execution: DBP dual buffers + FWP frozen window (TEST INFRASTRUCTURE).

Follows the paper's order step by step over W simulated workers:

* DBP: the Prefetch HBM Buffer for B_{t+1} is filled from the
  shard while B_t runs on the Active buffer, i.e. after write-back(t-1) and
  before update(t) (reading Q8); after update(t) the intersection
  K(B_t) & K(B_{t+1}) is copied Active -> Prefetch ("dual-buffer
  synchronization"); updated rows are written back; the
  buffer roles swap.
* FWP: B_t is split into N micro-batches (clustered or
  sequential); for each micro-batch the owners send the requested rows of the
  frozen Active buffer (re-sent per micro-batch), the source pools them,
  the gradients of that micro-batch's keys go back to the owners and are
  accumulated in (micro-batch, source) order; the update is applied
  once after micro-batch N.
* unsafe_six_stage: the refresh is skipped, reproducing the
  one-step asynchrony hazard (negative control).

Gradient sums are fp64 and rounded once at the update, like oracle.step; in
parity regime P1 (dyadic values) every sum is exact so the result must equal
oracle.step.sync_step bit for bit (Prop. 1, Prop. 2, Corollary 1: P:501-548).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence

import numpy as np

from . import cluster as C
from . import routing as R
from .step import LazyTable, bag_of_occurrence, sgd_rows


@dataclass
class Buffer:
    """HbmBuffer: rows for one step's owner-unique keys."""

    step: int
    keys: np.ndarray                    # ascending
    rows: np.ndarray                    # fp32 [len(keys), d]
    dirty: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))

    def index(self, keys):
        return np.searchsorted(self.keys, keys)


def dual_buffer_sync(active: Buffer, prefetch: Buffer) -> None:
    """prefetch.rows[k] := active.rows[k] for k in both key sets."""
    common = np.intersect1d(active.keys, prefetch.keys, assume_unique=True)
    if len(common):
        prefetch.rows[prefetch.index(common)] = active.rows[active.index(common)]


@dataclass
class PipeConfig:
    W: int
    N: int = 1
    cluster: str = "sequential"          # "sequential" | "clustered"
    pooling: str = "sum"
    grad_mode: str = "lin"               # "lin" | "quad"
    lr_over_B: float = 2.0 ** -10
    F: int = 1
    pipelined: bool = True               # prefetch(t+1) before update(t)
    unsafe_six_stage: bool = False
    optimizer: object = None             # None: SGD (Eq. 2); else step.RowwiseAdagrad


@dataclass
class StepTrace:
    pooled: List[List[np.ndarray]]       # [rank][mb] fp32, mb-local bag order
    perm: List[np.ndarray]
    mb_offsets: List[np.ndarray]
    table: Dict[int, np.ndarray]         # key -> row after the step (touched keys)


def _partition(cfg: PipeConfig, keys, offs):
    B = (len(offs) - 1) // cfg.F
    if cfg.cluster == "clustered":
        return C.cluster_rounds(C.sample_keysets(keys, offs, cfg.F), cfg.N)
    return C.cluster_sequential(B, cfg.N)


def _mb_bags(perm, mb_offsets, i, F):
    """Global bag indices of micro-batch i in mb-local order (p*F + f)."""
    samples = np.asarray(perm)[mb_offsets[i]:mb_offsets[i + 1]]
    return (samples[:, None] * F + np.arange(F)[None, :]).reshape(-1)


def nestpipe_train(shard_init: LazyTable, batches_by_step, douts_by_step,
                   cfg: PipeConfig) -> List[StepTrace]:
    """Run T steps of DBP+FWP over W simulated workers.

    batches_by_step[t][r] = (keys, bag_offsets) of rank r at step t;
    douts_by_step[t][r]   = fp32 dpooled in ORIGINAL bag order (LIN mode).
    """
    W, N, F = cfg.W, cfg.N, cfg.F
    T = len(batches_by_step)
    # per-owner host shards: one LazyTable each, holding only owned keys
    shards = [shard_init.copy() for _ in range(W)]

    def route(t):
        parts = [_partition(cfg, *batches_by_step[t][r]) for r in range(W)]
        mb_occ = [R.mb_of_occurrence(batches_by_step[t][r][1], F, *parts[r]) for r in range(W)]
        src, own = R.route_all(batches_by_step[t], W, mb_occ, N)
        return parts, src, own

    def retrieve(t, own):
        """Embedding Retrieval: owner o copies its requested rows."""
        bufs = []
        for o in range(W):
            keys = own[o].owner_keys
            if len(keys) and (R.shard_of(keys, W) != o).any():
                raise ValueError("foreign key at owner (shard violation, S:266)")
            bufs.append(Buffer(t, keys.copy(), shards[o].snapshot(keys)))
        return bufs

    traces: List[StepTrace] = []
    plan = route(0)
    active = retrieve(0, plan[2])
    for t in range(T):
        parts, src, own = plan
        nxt = None
        if t + 1 < T and cfg.pipelined:
            nxt_plan = route(t + 1)
            nxt = retrieve(t + 1, nxt_plan[2])       # shard state: after write-back(t-1)
        # ---------------- FWP frozen window over Active(t) ----------------
        acc = [np.zeros((len(active[o].keys), shard_init.dim), dtype=np.float64) for o in range(W)]
        pooled_all = [[None] * N for _ in range(W)]
        for i in range(N):
            # emb All2All: owner o sends rows of its send list (mb i, source s)
            for s in range(W):
                keys_s, offs_s = batches_by_step[t][s]
                rs = src[s]
                # rows the source receives for its mask-bit-i keys, owner-major
                sel = ((rs.mask >> i) & 1) == 1
                recv_keys = rs.uniq[sel]
                recv_rows = np.zeros((len(recv_keys), shard_init.dim), dtype=np.float32)
                for o in range(W):
                    lst = own[o].send_lists[i][s]
                    ks = own[o].recv_keys[lst]
                    rows = active[o].rows[own[o].owner_inv[lst]]
                    # positions of those keys among the source's mask-bit-i keys
                    seg = np.arange(rs.send_offsets[o], rs.send_offsets[o + 1])
                    seg = seg[((rs.mask[seg] >> i) & 1) == 1]
                    assert np.array_equal(rs.uniq[seg], ks)
                    recv_rows[rs.pos[i][seg]] = rows
                # pool / expand on the source (mb-local order)
                perm, mbo = parts[s]
                bags = _mb_bags(perm, mbo, i, F)
                offs_s = np.asarray(offs_s, dtype=np.int64)
                lens = offs_s[bags + 1] - offs_s[bags]
                occ = np.concatenate([np.arange(offs_s[b], offs_s[b + 1]) for b in bags]) \
                    if len(bags) else np.zeros(0, np.int64)
                rows_occ = recv_rows[rs.pos[i][rs.inverse[occ]]]
                if cfg.pooling == "sum":
                    mb_offs = np.concatenate([[0], np.cumsum(lens)])
                    acc64 = np.zeros((len(bags), shard_init.dim), dtype=np.float64)
                    np.add.at(acc64, bag_of_occurrence(mb_offs), rows_occ.astype(np.float64))
                    pooled = acc64.astype(np.float32)
                    dout = pooled if cfg.grad_mode == "quad" else \
                        np.asarray(douts_by_step[t][s])[bags]
                    contrib = np.asarray(dout, dtype=np.float64)[bag_of_occurrence(mb_offs)]
                else:
                    pooled = rows_occ.copy()
                    dout = pooled if cfg.grad_mode == "quad" else \
                        np.asarray(douts_by_step[t][s])[occ]
                    contrib = np.asarray(dout, dtype=np.float64)
                pooled_all[s][i] = pooled
                # source segment-sum per unique key of mb i, then grad All2All
                g_src = np.zeros((int(sel.sum()), shard_init.dim), dtype=np.float64)
                np.add.at(g_src, rs.pos[i][rs.inverse[occ]], contrib)
                for o in range(W):
                    seg = np.arange(rs.send_offsets[o], rs.send_offsets[o + 1])
                    seg = seg[((rs.mask[seg] >> i) & 1) == 1]
                    lst = own[o].send_lists[i][s]
                    # (micro-batch i, source s) order of accumulation
                    acc[o][own[o].owner_inv[lst]] += g_src[rs.pos[i][seg]]
        # ---------------- single deferred update + write-back ----------------
        for o in range(W):
            if len(active[o].keys):
                active[o].rows = sgd_rows(active[o].rows, acc[o], cfg.lr_over_B) if cfg.optimizer is None \
                    else cfg.optimizer.apply(active[o].keys, active[o].rows, acc[o])
                active[o].dirty = active[o].keys.copy()
                shards[o].set(active[o].keys, active[o].rows)
        table = {}
        for o in range(W):
            for k, row in zip(active[o].keys, active[o].rows):
                table[int(k)] = row.copy()
        traces.append(StepTrace(pooled_all, [p[0] for p in parts], [p[1] for p in parts], table))
        if t + 1 < T:
            if not cfg.pipelined:
                nxt_plan = route(t + 1)
                nxt = retrieve(t + 1, nxt_plan[2])
            if not cfg.unsafe_six_stage:
                for o in range(W):
                    dual_buffer_sync(active[o], nxt[o])
            active = nxt
            plan = nxt_plan
    return traces


def sync_train(table: LazyTable, batches_by_step, douts_by_step, lr_over_B,
               pooling="sum", grad_mode="lin", optimizer=None):
    """T steps of oracle.step.sync_step; returns per-step {key: row} of K(B_t)."""
    from .step import sync_step
    out = []
    for t, batches in enumerate(batches_by_step):
        res = sync_step(table, batches, douts_by_step[t] if douts_by_step else None,
                        lr_over_B, pooling, grad_mode, optimizer)
        rows = table.get(res.grads.keys)
        out.append({int(k): r.copy() for k, r in zip(res.grads.keys, rows)})
    return out


def first_divergence(traj_a: Sequence[Dict[int, np.ndarray]],
                     traj_b: Sequence[Dict[int, np.ndarray]], tol: float = 0.0):
    """compare_trajectories: first 1-based step whose rows differ
    by more than tol, or None."""
    for t, (a, b) in enumerate(zip(traj_a, traj_b)):
        keys = set(a) | set(b)
        for k in keys:
            if k not in a or k not in b:
                return t + 1
            if np.max(np.abs(a[k].astype(np.float64) - b[k].astype(np.float64))) > tol:
                return t + 1
    return None
