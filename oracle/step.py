"""The synchronous training step of Definition 1 / Eq. 1-2 (TEST INFRASTRUCTURE).

P:492-499 (Definition 1, Eq. 1: W_{t+1} = W_t - eta/|B_t| sum_xi grad F(W_t, xi)),
P:509-514 (Eq. 2: per key, e_k^{t+1} = e_k^t if k not in K(B_t), else
e_k^t - eta/|B_t| sum_xi grad_{e_k} F), S:282-290 (apply_sparse_grads),
S:353-361 (pool = element-wise sum of the sample's rows)
(scatter_embedding_grads: every key of a bag receives the bag's pooled grad).

Arithmetic (reading Q6): pooled sums and gradient sums are
accumulated in fp64 left to right (ascending global (rank, sample, feature,
position)) and rounded to fp32 once; the update is fp32(e - s*G) in fp64 with
s = lr_over_B as an fp32 value.  The step is computed over the global batch
with NO sharding: it is the plain definition that DBP/FWP must reproduce
(P:501-548).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Sequence, Tuple

import numpy as np

from . import prf


class LazyTable:
    """E_t over the whole vocabulary, materialised lazily:
    a key never written holds init_row(seed, key)."""

    def __init__(self, seed: int, dim: int, mode: str = "uniform"):
        self.seed, self.dim, self.mode = int(seed), int(dim), mode
        self.keys = np.zeros(0, dtype=np.int64)
        self.rows = np.zeros((0, dim), dtype=np.float32)

    def copy(self) -> "LazyTable":
        t = LazyTable(self.seed, self.dim, self.mode)
        t.keys, t.rows = self.keys.copy(), self.rows.copy()
        return t

    def _materialise(self, keys: np.ndarray) -> None:
        keys = np.unique(np.asarray(keys, dtype=np.int64))
        new = keys[~np.isin(keys, self.keys)]
        if len(new):
            allk = np.concatenate([self.keys, new])
            allr = np.concatenate([self.rows, prf.init_rows(self.seed, new, self.dim, self.mode)])
            order = np.argsort(allk, kind="stable")
            self.keys, self.rows = allk[order], allr[order]

    def get(self, keys) -> np.ndarray:
        keys = np.asarray(keys, dtype=np.int64)
        self._materialise(keys)
        return self.rows[np.searchsorted(self.keys, keys)]

    def set(self, keys, rows) -> None:
        keys = np.asarray(keys, dtype=np.int64)
        self._materialise(keys)
        self.rows[np.searchsorted(self.keys, keys)] = np.asarray(rows, dtype=np.float32)

    def snapshot(self, keys) -> np.ndarray:
        return self.get(keys).copy()


def bag_of_occurrence(bag_offsets) -> np.ndarray:
    bag_offsets = np.asarray(bag_offsets, dtype=np.int64)
    return np.repeat(np.arange(len(bag_offsets) - 1), np.diff(bag_offsets))


def pool_sum(rows_of_occ: np.ndarray, bag_offsets) -> np.ndarray:
    """pooled[bag] = sum of its rows, fp64 left to right, one rounding.
    An empty bag pools to the zero vector (reading Q5)."""
    bag_offsets = np.asarray(bag_offsets, dtype=np.int64)
    nb = len(bag_offsets) - 1
    acc = np.zeros((nb, rows_of_occ.shape[1]), dtype=np.float64)
    np.add.at(acc, bag_of_occurrence(bag_offsets), rows_of_occ.astype(np.float64))
    return acc.astype(np.float32)


def forward(table: LazyTable, keys, bag_offsets, pooling: str = "sum") -> np.ndarray:
    """Forward lookup of one rank's batch against E_t (each source
    'obtains the complete set of embedding vectors required by its batch')."""
    rows = table.get(keys)
    if pooling == "sum":
        return pool_sum(rows, bag_offsets)
    if pooling == "none":
        return rows.astype(np.float32).copy()
    raise ValueError(pooling)


@dataclass
class KeyGrads:
    keys: np.ndarray    # int64[U]: K(B_t), ascending
    grad: np.ndarray    # fp64[U, d]: sum of contributions
    absgrad: np.ndarray  # fp64[U, d]: sum of |contributions| (tolerance scale)
    count: np.ndarray   # int64[U]: number of contributions


def key_grads(batches: Sequence[Tuple[np.ndarray, np.ndarray]],
              douts: Sequence[np.ndarray], pooling: str = "sum") -> KeyGrads:
    """Eq. 2 second case + S:383-391: the sum over all occurrences of key k in
    the GLOBAL batch (ranks in order = contiguous sample slices) of the
    gradient of the bag (pooled) or occurrence (unpooled) it sits in."""
    all_keys, contribs = [], []
    for (keys, offs), dout in zip(batches, douts):
        keys = np.asarray(keys, dtype=np.int64)
        all_keys.append(keys)
        if pooling == "sum":
            contribs.append(np.asarray(dout, dtype=np.float64)[bag_of_occurrence(offs)])
        else:
            contribs.append(np.asarray(dout, dtype=np.float64))
    keys = np.concatenate(all_keys)
    d = douts[0].shape[1]
    c = np.concatenate(contribs) if len(contribs) else np.zeros((0, d))
    uk, inv = np.unique(keys, return_inverse=True)
    g = np.zeros((len(uk), d), dtype=np.float64)
    a = np.zeros((len(uk), d), dtype=np.float64)
    np.add.at(g, inv, c)
    np.add.at(a, inv, np.abs(c))
    cnt = np.bincount(inv, minlength=len(uk)).astype(np.int64)
    return KeyGrads(uk, g, a, cnt)


def sgd_rows(rows: np.ndarray, grad: np.ndarray, lr_over_B: float) -> np.ndarray:
    """Eq. 2 / S:282-290: e' = e - (eta/|B|) * sum, one rounding to fp32."""
    s = np.float64(np.float32(lr_over_B))
    return (rows.astype(np.float64) - s * grad).astype(np.float32)


class RowwiseAdagrad:
    """Row-wise AdaGrad, the sparse optimizer of SURVEY §8(f) NEXT-2 (the paper
    and SPEC leave the optimizer open; industry convention = FBGEMM's
    exact row-wise AdaGrad).  One accumulator m per embedding row, initially
    `init`; for a key k of K(B_t) with summed gradient G_k (the same sum Eq. 2
    scales):
        g   = grad_scale * G_k                      (grad_scale = 1/|B|)
        m_k = m_k + (1/d) * sum_j g_j^2
        e_k = e_k - lr * g / (sqrt(m_k) + eps)
    Rows of keys outside K(B_t) and their accumulators are unchanged.  fp64
    arithmetic on the fp32 inputs (grad_scale, lr, eps as fp32 values), the row
    rounded to fp32 once per step; the accumulator is kept in fp64.
    """

    def __init__(self, lr: float, grad_scale: float, eps: float = 1e-8, init: float = 0.0):
        self.lr = np.float64(np.float32(lr))
        self.gs = np.float64(np.float32(grad_scale))
        self.eps = np.float64(np.float32(eps))
        self.init = float(init)
        self.state = {}

    def get_state(self, keys) -> np.ndarray:
        return np.array([self.state.get(int(k), self.init) for k in np.asarray(keys, np.int64)], np.float64)

    def apply(self, keys, rows: np.ndarray, grad: np.ndarray) -> np.ndarray:
        keys = np.asarray(keys, np.int64)
        g = self.gs * np.asarray(grad, np.float64)
        m = self.get_state(keys) + (g * g).mean(axis=1)
        for k, mk in zip(keys, m):
            self.state[int(k)] = float(mk)
        mult = self.lr / (np.sqrt(m) + self.eps)
        return (rows.astype(np.float64) - mult[:, None] * g).astype(np.float32)


@dataclass
class StepResult:
    pooled: List[np.ndarray]   # per rank, fp32
    grads: KeyGrads


def sync_step(table: LazyTable, batches, douts=None, lr_over_B: float = 2.0 ** -10,
              pooling: str = "sum", grad_mode: str = "lin", optimizer=None) -> StepResult:
    """oracle.sync_step: one synchronous step over the global batch.

    grad_mode 'lin'  : dpooled = douts[r] (seeded, independent of E)
    grad_mode 'quad' : L = 1/2 sum ||pooled||^2, so dpooled = pooled.
    Mutates `table` to E_{t+1}; only keys in K(B_t) change (Eq. 2).
    optimizer: None = SGD of Eq. 2 with lr_over_B, else a RowwiseAdagrad.
    """
    pooled = [forward(table, k, o, pooling) for (k, o) in batches]
    if grad_mode == "quad":
        douts = pooled
    g = key_grads(batches, douts, pooling)
    if len(g.keys):
        rows = table.get(g.keys)
        new = sgd_rows(rows, g.grad, lr_over_B) if optimizer is None else optimizer.apply(g.keys, rows, g.grad)
        table.set(g.keys, new)
    return StepResult(pooled, g)
