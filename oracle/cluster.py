"""Key-centric sample clustering for FWP (TEST INFRASTRUCTURE).

P:470-482 ("group samples that share more sparse keys into the same
micro-batch, maximizing key redundancy within micro-batch"; it "only changes
the order of embedding and gradient communication").  The paper states only
the objective; S:544-552 / S:590 fix a sequential greedy, SURVEY §8(c) "Clustering
spec" fixes the round-based parallel greedy that the CUDA path implements
(reading R-CLUSTER).  All three modes return (perm, mb_offsets): micro-batch
i is the samples perm[mb_offsets[i]:mb_offsets[i+1]], equal sizes.
"""
from __future__ import annotations

import itertools
from typing import List, Sequence, Tuple

import numpy as np


def sample_keysets(keys, bag_offsets, F: int) -> List[np.ndarray]:
    """Distinct packed keys of every sample (S:565 'a sample's key set')."""
    keys = np.asarray(keys, dtype=np.int64)
    offs = np.asarray(bag_offsets, dtype=np.int64)
    B = (len(offs) - 1) // F
    return [np.unique(keys[offs[b * F]:offs[(b + 1) * F]]) for b in range(B)]


def partition_cost(keysets: Sequence[np.ndarray], perm, mb_offsets) -> int:
    """sum_i |K(M_i)|: keys sent over all micro-batches."""
    tot = 0
    for i in range(len(mb_offsets) - 1):
        mem = [keysets[s] for s in perm[mb_offsets[i]:mb_offsets[i + 1]]]
        tot += len(np.unique(np.concatenate(mem))) if mem else 0
    return tot


def _check(B: int, N: int) -> int:
    if N < 1 or B % N != 0:
        raise ValueError("batch size must be divisible by the micro-batch count (S:548)")
    return B // N


def cluster_sequential(B: int, N: int):
    """Mode 'sequential': slice by ascending sample id."""
    cap = _check(B, N)
    return np.arange(B, dtype=np.int64), np.arange(N + 1, dtype=np.int64) * cap


def admission_sizes(cap: int, max_rounds: int = 10_000):
    """q_r of the round schedule: Q_0 = 2^32, Q_r = floor(5 Q_{r-1} / 4),
    q_r = max(1, Q_r >> 32) (exact u64 fixed point)."""
    Q = 1 << 32
    for _ in range(max_rounds):
        if Q < (1 << 62):
            Q = (5 * Q) // 4
        yield max(1, Q >> 32)


def cluster_rounds(keysets: Sequence[np.ndarray], N: int):
    """Mode 'clustered': the round-based parallel greedy of SURVEY §8(c).

    Seeds: g=0 takes the largest sample (ties: lowest id); g>0 takes the
    unassigned sample maximising (-|keys(s) & union of earlier seeds|, size, -id).
    Round r: snapshot S[s][g] = |keys(s) & union(g)| for unassigned s; for
    g = 0..N-1 in order take min(cap - have_g, q_r) samples not yet taken, ranked
    by S[s][g] desc, (size - S[s][g]) asc, id asc; unions grow after the round.
    """
    B = len(keysets)
    cap = _check(B, N)
    if N == 1:
        return cluster_sequential(B, N)
    size = np.array([len(k) for k in keysets], dtype=np.int64)
    ids = np.arange(B, dtype=np.int64)
    group = np.full(B, -1, dtype=np.int64)
    # key -> bitmask of groups whose union contains it
    allk = np.unique(np.concatenate(keysets)) if B else np.zeros(0, np.int64)
    kidx = [np.searchsorted(allk, k) for k in keysets]
    flat = np.concatenate(kidx) if B else np.zeros(0, np.int64)
    owner_s = np.repeat(ids, size)
    inmask = np.zeros(len(allk), dtype=np.int64)

    # seeds
    seed_union = np.zeros(len(allk), dtype=bool)
    for g in range(N):
        un = group < 0
        ov = np.zeros(B, dtype=np.int64)
        np.add.at(ov, owner_s, seed_union[flat].astype(np.int64))
        cand = ids[un]
        order = np.lexsort((cand, -size[cand], ov[cand]))   # ov asc, size desc, id asc
        s = cand[order[0]]
        group[s] = g
        seed_union[kidx[s]] = True
        inmask[kidx[s]] |= (1 << g)
    have = np.ones(N, dtype=np.int64)

    for q in admission_sizes(cap):
        if (group >= 0).all():
            break
        # snapshot S[s][g]
        S = np.zeros((N, B), dtype=np.int64)
        for g in range(N):
            np.add.at(S[g], owner_s, (inmask[flat] >> g) & 1)
        taken = group >= 0
        new_members = []
        for g in range(N):
            take = int(min(cap - have[g], q))
            if take <= 0:
                new_members.append(np.zeros(0, np.int64))
                continue
            cand = ids[~taken]
            Sg = S[g][cand]
            order = np.lexsort((cand, size[cand] - Sg, -Sg))
            chosen = cand[order[:take]]
            group[chosen] = g
            taken[chosen] = True
            have[g] += len(chosen)
            new_members.append(chosen)
        for g in range(N):
            for s in new_members[g]:
                inmask[kidx[s]] |= (1 << g)
    perm = np.lexsort((ids, group))
    return perm.astype(np.int64), np.arange(N + 1, dtype=np.int64) * cap


def cluster_spec_greedy(keysets: Sequence[np.ndarray], N: int):
    """S:590 sequential greedy (quality reference, small inputs only): open a
    group with the largest unassigned sample (ties: lowest id), fill it to cap
    with the unassigned sample of maximal |intersection| with the group union
    (ties: smaller union growth, then lowest id)."""
    B = len(keysets)
    cap = _check(B, N)
    sets = [set(int(x) for x in k) for k in keysets]
    unassigned = set(range(B))
    groups = []
    for _ in range(N):
        s0 = min(unassigned, key=lambda s: (-len(sets[s]), s))
        unassigned.remove(s0)
        members, union = [s0], set(sets[s0])
        while len(members) < cap:
            s = min(unassigned, key=lambda s: (-len(sets[s] & union),
                                               len(sets[s] - union), s))
            unassigned.remove(s)
            members.append(s)
            union |= sets[s]
        groups.append(sorted(members))
    perm = np.array([s for g in groups for s in g], dtype=np.int64)
    return perm, np.arange(N + 1, dtype=np.int64) * cap


def brute_force_best(keysets: Sequence[np.ndarray], N: int) -> int:
    """Minimum of sum_i |K(M_i)| over all balanced partitions (tiny B only)."""
    B = len(keysets)
    cap = _check(B, N)
    best = None

    def rec(remaining, acc):
        nonlocal best
        if not remaining:
            best = acc if best is None else min(best, acc)
            return
        first = remaining[0]
        for rest in itertools.combinations(remaining[1:], cap - 1):
            grp = (first,) + rest
            cost = len(set().union(*[set(int(x) for x in keysets[s]) for s in grp]))
            rec([s for s in remaining if s not in grp], acc + cost)

    rec(list(range(B)), 0)
    return int(best)


def mb_of_sample(perm, mb_offsets, B: int) -> np.ndarray:
    out = np.full(B, -1, dtype=np.int64)
    for i in range(len(mb_offsets) - 1):
        out[np.asarray(perm)[mb_offsets[i]:mb_offsets[i + 1]]] = i
    return out
