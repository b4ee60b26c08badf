"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no routing, pooling, gradient
or update math).  It only draws the random inputs both sides consume:

* batches of packed sparse keys in CSR form (``keys`` int64[K] and
  ``bag_offsets`` int32[B*F+1], sample-major: bag index = b*F + f),
* the synthetic loss gradients ``dout`` of SURVEY.md §8(c) O5 (mode LIN),
* the workload configurations of BASELINE.json ``configs``.

Key packing: ``key = (table << 40) | row`` with
``row < rows[table]``.  Popularity is a bounded Zipf over ranks with an affine
rank->row bijection; the paper only says accesses are
"highly skewed" (§IV-A).

Recipes are documented in DESIGN.md ("Input recipe").
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from typing import List, Tuple

import numpy as np

ROW_BITS = 40
ROW_MASK = (1 << ROW_BITS) - 1


@dataclass(frozen=True)
class WorkloadConfig:
    """One synthetic workload (BASELINE.json ``configs``)."""

    name: str
    table_rows: Tuple[int, ...]
    dim: int
    batch_local: int              # samples per rank (per GPU)
    bag_len: Tuple[int, int]      # inclusive uniform range of keys per bag
    bag_repeats: bool             # may a bag repeat a key
    zipf: float
    pooling: str = "sum"          # "sum" (pooled) or "none" (unpooled expand)
    world: int = 1                # default number of shards
    micro_batches: int = 1        # default FWP N
    tower_layers: int = 4         # stand-in tower depth (timing only)
    tower_hidden: int = 1024
    feature_table: Tuple[int, ...] = ()   # table of every feature (default: feature f -> table f)

    @property
    def num_tables(self) -> int:
        return len(self.table_rows)

    @property
    def num_features(self) -> int:
        return len(self.feature_table) if self.feature_table else len(self.table_rows)

    def table_of_feature(self, f: int) -> int:
        return self.feature_table[f] if self.feature_table else f

    def with_(self, **kw) -> "WorkloadConfig":
        return replace(self, **kw)


def _geomspace_rows(lo: int, hi: int, n: int) -> Tuple[int, ...]:
    return tuple(int(round(x)) for x in np.geomspace(lo, hi, n))


CONFIGS = {
    # BASELINE.json configs[0]: 4 tables x 1,000 rows, dim 16, global batch 64
    # (32 per shard at W=2), 1-3 keys/bag without repeats, Zipf 1.05
    "tiny": WorkloadConfig("tiny", (1000,) * 4, 16, 32, (1, 3), False, 1.05,
                           world=2),
    # configs[1]: 26 tables, 1M-10M rows, dim 128 fp32, batch 65,536/GPU, sum
    "dlrm": WorkloadConfig("dlrm", _geomspace_rows(1_000_000, 10_000_000, 26),
                           128, 65536, (1, 3), True, 1.05, world=8,
                           micro_batches=4),
    # configs[2]: 8 tables x 50M rows, dim 64, batch 8,192, seq 1,024 unpooled
    "genrec": WorkloadConfig("genrec", (50_000_000,) * 8, 64, 8192,
                             (1024, 1024), True, 1.2, pooling="none", world=8),
    # configs[3]: 1 table x 100M rows, dim 128, 26 bags per sample
    "dbp_stress": WorkloadConfig("dbp_stress", (100_000_000,), 128, 65536,
                                 (1, 3), True, 1.05, world=8, feature_table=(0,) * 26),
}


# ----------------------------------------------------------------------------
# random streams
# ----------------------------------------------------------------------------

def rng_for(seed: int, *stream: int) -> np.random.Generator:
    """Independent, reproducible stream per (seed, purpose...)."""
    return np.random.default_rng(np.random.SeedSequence([int(seed) & 0xFFFFFFFF,
                                                         *[int(s) for s in stream]]))


def zipf_ranks(rng: np.random.Generator, s: float, n: int, size: int) -> np.ndarray:
    """Bounded Zipf(s) ranks in [0, n) by the continuous inverse CDF.

    Density proportional to x^-s on [1, n+1); rank = floor(x) - 1.
    """
    u = rng.random(size)
    if abs(s - 1.0) < 1e-12:
        x = np.exp(u * math.log(n + 1.0))
    else:
        a = 1.0 - s
        top = (n + 1.0) ** a
        x = (1.0 + u * (top - 1.0)) ** (1.0 / a)
    r = np.floor(x).astype(np.int64) - 1
    return np.clip(r, 0, n - 1)


def rank_to_row_params(rows: int, salt: int) -> Tuple[int, int]:
    """Affine bijection rank -> (a*rank + c) mod rows."""
    a = 2_654_435_761
    if a % 2 == 0:
        a += 1
    while math.gcd(a, rows) != 1:
        a += 2
    c = (salt * 0x9E3779B1 + 12345) % rows
    return a % rows if rows > 1 else 0, c


def ranks_to_rows(ranks: np.ndarray, rows: int, salt: int) -> np.ndarray:
    if rows == 1:
        return np.zeros_like(ranks)
    a, c = rank_to_row_params(rows, salt)
    # a < rows <= 2^31 and ranks < rows, so a*rank < 2^62: no overflow
    return (ranks.astype(np.int64) * np.int64(a) + np.int64(c)) % np.int64(rows)


def pack_keys(table: np.ndarray | int, rows: np.ndarray) -> np.ndarray:
    return (np.int64(table) << np.int64(ROW_BITS)) | rows.astype(np.int64)


def unpack_keys(keys: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    keys = np.asarray(keys, dtype=np.int64)
    return keys >> ROW_BITS, keys & ROW_MASK


# ----------------------------------------------------------------------------
# batches
# ----------------------------------------------------------------------------

def _draw_table_keys(rng, cfg: WorkloadConfig, f: int, lengths: np.ndarray,
                     salt: int) -> np.ndarray:
    """Rows for every bag of feature f, concatenated in bag order."""
    tab = cfg.table_of_feature(f)
    rows_t = cfg.table_rows[tab]
    n = int(lengths.sum())
    ranks = zipf_ranks(rng, cfg.zipf, rows_t, n)
    if not cfg.bag_repeats:
        # redraw any key that repeats inside its bag
        starts = np.concatenate([[0], np.cumsum(lengths)[:-1]])
        bag_id = np.repeat(np.arange(len(lengths)), lengths)
        for _ in range(1000):
            order = np.lexsort((ranks, bag_id))
            sb, sr = bag_id[order], ranks[order]
            dup_sorted = np.zeros(n, dtype=bool)
            dup_sorted[1:] = (sb[1:] == sb[:-1]) & (sr[1:] == sr[:-1])
            if not dup_sorted.any():
                break
            idx = order[dup_sorted]
            ranks[idx] = zipf_ranks(rng, cfg.zipf, rows_t, len(idx))
        else:  # pragma: no cover
            raise RuntimeError("could not draw distinct bag keys")
        del starts
    return pack_keys(tab, ranks_to_rows(ranks, rows_t, salt=tab + 1))


def gen_batch(cfg: WorkloadConfig, seed: int, step: int, rank: int,
              batch: int | None = None) -> Tuple[np.ndarray, np.ndarray]:
    """One rank's local batch: (keys int64[K], bag_offsets int32[B*F+1]).

    Sample-major CSR: bag (b, f) = b*F + f holds keys of table f for sample b.
    """
    B = cfg.batch_local if batch is None else batch
    F = cfg.num_features
    rng = rng_for(seed, 1, step, rank)
    lo, hi = cfg.bag_len
    lengths = rng.integers(lo, hi + 1, size=(B, F)).astype(np.int64)
    bag_offsets = np.zeros(B * F + 1, dtype=np.int64)
    np.cumsum(lengths.reshape(-1), out=bag_offsets[1:])
    keys = np.empty(int(bag_offsets[-1]), dtype=np.int64)
    for f in range(F):
        tk = _draw_table_keys(rng_for(seed, 2, step, rank, f), cfg, f,
                              lengths[:, f], salt=f)
        # scatter table-f keys into their bags
        starts = bag_offsets[np.arange(B) * F + f]
        ln = lengths[:, f]
        dst = np.repeat(starts, ln) + (np.arange(int(ln.sum()))
                                       - np.repeat(np.cumsum(ln) - ln, ln))
        keys[dst] = tk
    assert bag_offsets[-1] < 2**31
    return keys, bag_offsets.astype(np.int32)


def gen_global_batch(cfg: WorkloadConfig, seed: int, step: int, world: int):
    """Per-rank batches for all ranks; rank r owns the contiguous slice r."""
    return [gen_batch(cfg, seed, step, r) for r in range(world)]


def gen_dout(seed: int, step: int, rank: int, n_rows: int, dim: int,
             mode: str = "dyadic", mb: int = 0) -> np.ndarray:
    """Synthetic loss gradient R[t, b, f, :] (SURVEY §8(c) O5 mode LIN).

    dyadic: integers in [-4, 4] times 2^-8 (exact in fp32; parity regime P1);
    realistic: standard normal fp32 (parity regime P2).
    """
    rng = rng_for(seed, 3, step, rank, mb)
    if mode == "dyadic":
        return (rng.integers(-4, 5, size=(n_rows, dim)).astype(np.float32)
                * np.float32(2.0 ** -8))
    if mode == "realistic":
        return rng.standard_normal((n_rows, dim), dtype=np.float32)
    raise ValueError(mode)


def gen_overlap_batches(cfg: WorkloadConfig, seed: int, steps: int, rank: int,
                        p_reuse: float) -> List[Tuple[np.ndarray, np.ndarray]]:
    """DBP stress (BASELINE configs[3]): batch t+1 keeps the bag structure of a
    fresh draw and reuses, per key slot, the key of batch t at the same slot
    with probability p_reuse (when the slot exists and holds the same table),
    else keeps the fresh Zipf key."""
    out = [gen_batch(cfg, seed, 0, rank)]
    for t in range(1, steps):
        prev, _ = out[-1]
        fresh, offs = gen_batch(cfg, seed, t, rank)
        rng = rng_for(seed, 4, t, rank)
        n = min(len(prev), len(fresh))
        take = (rng.random(n) < p_reuse) & ((prev[:n] >> ROW_BITS) == (fresh[:n] >> ROW_BITS))
        nk = fresh.copy()
        nk[:n][take] = prev[:n][take]
        out.append((nk, offs))
    return out


def gen_correlated_batch(cfg: WorkloadConfig, seed: int, step: int, rank: int,
                         groups: int = 64, rho: float = 0.5,
                         batch: int | None = None):
    """FWP sweep correlated variant: every sample belongs to
    one of `groups` latent groups; with probability rho a key is drawn through
    the group's private rank->row permutation, else through the global one."""
    B = cfg.batch_local if batch is None else batch
    F = cfg.num_features
    rng = rng_for(seed, 5, step, rank)
    lo, hi = cfg.bag_len
    lengths = rng.integers(lo, hi + 1, size=(B, F)).astype(np.int64)
    grp = rng.integers(0, groups, size=B)
    bag_offsets = np.zeros(B * F + 1, dtype=np.int64)
    np.cumsum(lengths.reshape(-1), out=bag_offsets[1:])
    keys = np.empty(int(bag_offsets[-1]), dtype=np.int64)
    for f in range(F):
        tab = cfg.table_of_feature(f)
        rows_t = cfg.table_rows[tab]
        ln = lengths[:, f]
        n = int(ln.sum())
        r2 = rng_for(seed, 6, step, rank, f)
        ranks = zipf_ranks(r2, cfg.zipf, rows_t, n)
        g_of = np.repeat(grp, ln)
        private = r2.random(n) < rho
        rows = ranks_to_rows(ranks, rows_t, salt=f)
        for g in np.unique(g_of[private]):
            sel = private & (g_of == g)
            rows[sel] = ranks_to_rows(ranks[sel], rows_t, salt=f + 1000 * (1 + int(g)))
        starts = bag_offsets[np.arange(B) * F + f]
        dst = np.repeat(starts, ln) + (np.arange(n) - np.repeat(np.cumsum(ln) - ln, ln))
        keys[dst] = pack_keys(tab, rows)
    return keys, bag_offsets.astype(np.int32)
