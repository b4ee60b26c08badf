"""Key routing of the DBP Key-Routing / Embedding-Retrieval stages (TEST INFRASTRUCTURE).

P:343 ("sparse keys within the batch are first deduplicated ... then partitioned
into buckets based on embedding table sharding rules ... routed to destination
workers ... via All2All"), P:347 ("each destination worker again performs
sparse key deduplication"), S:164-172 (all_to_all delivery order)
(shard_of, dedup), S:460-468 (stage_key_routing)
(microbatch_routing: dedup within the micro-batch only).

Readings: keys are packed (table << 40) | row (Q2); the sharding
rule is owner = row mod W, local row = row div W (Q1); the
source's unique list is ordered by (owner, key) ascending, the owner's list by
key ascending, receives concatenate sources in ascending rank (Q3).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List

import numpy as np

ROW_BITS = 40
ROW_MASK = (1 << ROW_BITS) - 1


def table_of(keys) -> np.ndarray:
    return np.asarray(keys, dtype=np.int64) >> ROW_BITS


def row_of(keys) -> np.ndarray:
    return np.asarray(keys, dtype=np.int64) & ROW_MASK


def shard_of(keys, W: int) -> np.ndarray:
    """owner worker of each key = row mod W (reading Q1)."""
    return row_of(keys) % W


def local_row(keys, W: int) -> np.ndarray:
    """Row index inside the owner's shard of the key's table: row div W."""
    return row_of(keys) // W


def dedup(keys):
    """(unique ascending, inverse) with unique[inverse] == keys."""
    keys = np.asarray(keys, dtype=np.int64)
    return np.unique(keys, return_inverse=True)


def mb_of_occurrence(bag_offsets, F: int, perm, mb_offsets) -> np.ndarray:
    """Micro-batch index of every key occurrence (S:38-41 MicroBatch).

    Micro-batch i holds the samples perm[mb_offsets[i] : mb_offsets[i+1]].
    """
    bag_offsets = np.asarray(bag_offsets, dtype=np.int64)
    B = (len(bag_offsets) - 1) // F
    mb_of_sample = np.empty(B, dtype=np.int64)
    for i in range(len(mb_offsets) - 1):
        mb_of_sample[np.asarray(perm)[mb_offsets[i]:mb_offsets[i + 1]]] = i
    lens = np.diff(bag_offsets)
    sample_of_bag = np.arange(B * F) // F
    return np.repeat(mb_of_sample[sample_of_bag], lens)


@dataclass
class SourceRoute:
    """What one source worker computes in Key Routing."""

    uniq: np.ndarray          # int64[U_s]: unique keys, (owner, key) ascending
    inverse: np.ndarray       # int64[K]: uniq[inverse] == keys
    send_counts: np.ndarray   # int64[W]
    send_offsets: np.ndarray  # int64[W+1]
    mask: np.ndarray          # int64[U_s]: bit i set iff key occurs in micro-batch i
    mb_counts: np.ndarray     # int64[N, W]: keys of micro-batch i sent to owner o
    pos: np.ndarray           # int64[N, U_s]: index of uniq[u] among mask-bit-i keys


def route_source(keys, W: int, mb_occ=None, N: int = 1) -> SourceRoute:
    """Source-side dedup + bucketing.

    uniq is sorted by (shard_of, key); inverse maps each occurrence to its
    unique slot; send_counts/offsets bucket uniq per owner; mask records the
    micro-batches a key occurs in (per-micro-batch dedup scope).
    """
    keys = np.asarray(keys, dtype=np.int64)
    if mb_occ is None:
        mb_occ = np.zeros(len(keys), dtype=np.int64)
    u, inv = dedup(keys)
    owner = shard_of(u, W)
    order = np.lexsort((u, owner))          # primary owner, secondary key
    uniq = u[order]
    slot = np.empty(len(order), dtype=np.int64)
    slot[order] = np.arange(len(order))
    inverse = slot[inv] if len(keys) else np.zeros(0, dtype=np.int64)
    send_counts = np.bincount(shard_of(uniq, W), minlength=W).astype(np.int64)
    send_offsets = np.concatenate([[0], np.cumsum(send_counts)]).astype(np.int64)
    mask = np.zeros(len(uniq), dtype=np.int64)
    np.bitwise_or.at(mask, inverse, np.left_shift(1, np.asarray(mb_occ, dtype=np.int64)))
    mb_counts = np.zeros((N, W), dtype=np.int64)
    pos = np.zeros((N, len(uniq)), dtype=np.int64)
    for i in range(N):
        has = ((mask >> i) & 1).astype(np.int64)
        pos[i] = np.cumsum(has) - has
        for o in range(W):
            mb_counts[i, o] = has[send_offsets[o]:send_offsets[o + 1]].sum()
    return SourceRoute(uniq, inverse, send_counts, send_offsets, mask, mb_counts, pos)


def all_to_all(payloads: List[List[np.ndarray]]) -> List[List[np.ndarray]]:
    """payloads[s][r] is what sender s addresses to receiver r;
    receiver r gets [payloads[0][r], ..., payloads[W-1][r]] (ascending source)."""
    W = len(payloads)
    for p in payloads:
        if len(p) != W:
            raise ValueError("payload must have W destination lists")
    return [[payloads[s][r] for s in range(W)] for r in range(W)]


@dataclass
class OwnerRoute:
    """What one owner computes in Embedding Retrieval."""

    recv_keys: np.ndarray     # int64[R_o]: received keys, sources concatenated
    recv_mask: np.ndarray     # int64[R_o]
    recv_offsets: np.ndarray  # int64[W+1]: source segments of recv_keys
    owner_keys: np.ndarray    # int64[U_o]: unique, ascending
    owner_inv: np.ndarray     # int64[R_o]: owner_keys[owner_inv] == recv_keys
    send_lists: list          # [N][W] arrays of recv positions requested in mb i


def route_owner(recv_keys_by_src: List[np.ndarray], recv_mask_by_src: List[np.ndarray],
                N: int = 1) -> OwnerRoute:
    """Owner-side second dedup across sources and the per
    (micro-batch, source) send lists (keys of micro-batch i are
    re-sent in every micro-batch that uses them, in the order the source sent)."""
    W = len(recv_keys_by_src)
    recv_keys = np.concatenate([np.asarray(k, dtype=np.int64) for k in recv_keys_by_src]) \
        if W else np.zeros(0, np.int64)
    recv_mask = np.concatenate([np.asarray(m, dtype=np.int64) for m in recv_mask_by_src]) \
        if W else np.zeros(0, np.int64)
    counts = [len(k) for k in recv_keys_by_src]
    recv_offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    owner_keys, owner_inv = dedup(recv_keys)
    send_lists = []
    for i in range(N):
        per_src = []
        for s in range(W):
            r = np.arange(recv_offsets[s], recv_offsets[s + 1])
            per_src.append(r[((recv_mask[r] >> i) & 1) == 1])
        send_lists.append(per_src)
    return OwnerRoute(recv_keys, recv_mask, recv_offsets, owner_keys, owner_inv, send_lists)


def route_all(batches, W: int, mb_occ_list=None, N: int = 1):
    """Full Key Routing over W simulated workers: returns
    (source routes, owner routes)."""
    if mb_occ_list is None:
        mb_occ_list = [None] * W
    src = [route_source(batches[r][0], W, mb_occ_list[r], N) for r in range(W)]
    payload_keys = [[s.uniq[s.send_offsets[o]:s.send_offsets[o + 1]] for o in range(W)]
                    for s in src]
    payload_mask = [[s.mask[s.send_offsets[o]:s.send_offsets[o + 1]] for o in range(W)]
                    for s in src]
    recv_k = all_to_all(payload_keys)
    recv_m = all_to_all(payload_mask)
    own = [route_owner(recv_k[o], recv_m[o], N) for o in range(W)]
    return src, own
