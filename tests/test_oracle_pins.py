"""Pins of the CPU oracle against things other than itself (-m "not gpu").

Every oracle function is checked against worked examples printed in SPEC.md
(tests/golden/spec_examples.json, each cited), closed forms, brute force on
tiny inputs, or invariants the paper states.
"""
import json
import os
from fractions import Fraction
import itertools

import numpy as np
import pytest

import workload as WL
from oracle import cluster as C
from oracle import pipeline as P
from oracle import prf, routing as R, step as S

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# ----------------------------------------------------------------------------- prf
def test_splitmix64_reference_vectors():
    for x, y in GOLD["splitmix64"]["cases"]:
        x = int(x, 16) if isinstance(x, str) else x
        got = int(prf.splitmix64(np.array([x], dtype=np.uint64))[0])
        assert got == int(y, 16)


def test_init_rows_deterministic_and_seeded():
    keys = np.array([3, 7, (2 << 40) | 11], dtype=np.int64)
    a = prf.init_rows(1, keys, 16)
    assert np.array_equal(a, prf.init_rows(1, keys, 16))
    assert not np.array_equal(a, prf.init_rows(2, keys, 16))
    # a row depends only on (seed, key, j): order/batching independent
    assert np.array_equal(prf.init_rows(1, keys[::-1], 16), a[::-1])


def test_init_rows_range_and_moments():
    d = 16
    v = prf.init_rows(5, np.arange(10000), d).astype(np.float64).ravel()
    lim = 1 / np.sqrt(d)
    assert v.min() >= -lim - 1e-7 and v.max() < lim
    # uniform on [-lim, lim): mean 0, var lim^2/3; 3-sigma Monte Carlo
    n = len(v)
    assert abs(v.mean()) < 3 * lim / np.sqrt(3 * n)
    assert abs(v.var() - lim ** 2 / 3) < 0.02 * lim ** 2


def test_init_rows_single_rounding_exact():
    """v must be the correctly rounded value of lo + scale*u (what fmaf gives),
    checked with exact rational arithmetic."""
    d = 128
    keys = np.arange(50)
    h = prf.prf_words(9, keys, d)
    v = prf.init_rows(9, keys, d)
    lo = Fraction(float(np.float32(-1.0 / np.sqrt(d))))
    sc = Fraction(float(np.float32(2.0 / np.sqrt(d))))
    for i in range(0, 50, 7):
        for j in range(0, d, 13):
            u = Fraction(int(h[i, j]) >> 40, 1 << 24)
            exact = lo + sc * u
            # round-to-nearest fp32 of the exact rational
            f = np.float32(float(exact))
            cands = [np.nextafter(f, np.float32(-1)), f, np.nextafter(f, np.float32(1))]
            best = min(cands, key=lambda c: abs(Fraction(float(c)) - exact))
            assert v[i, j] == best


def test_init_rows_dyadic_values():
    v = prf.init_rows(3, np.arange(4000), 8, "dyadic").ravel() * 256
    assert np.array_equal(v, np.round(v)) and v.min() == -8 and v.max() == 7
    counts = np.bincount((v + 8).astype(int), minlength=16)
    assert counts.min() > 0.8 * len(v) / 16


# ----------------------------------------------------------------------------- routing
def test_spec_dedup_and_shard_examples():
    for c in GOLD["dedup"]["cases"]:
        u, inv = R.dedup(np.array(c["keys"], dtype=np.int64))
        assert u.tolist() == c["unique"] and inv.tolist() == c["inverse"]
    for k, W, o in GOLD["shard_of"]["cases"]:
        assert int(R.shard_of(np.array([k]), W)[0]) == o
    for a, b in GOLD["canonical_key_order"]["cases"]:
        assert R.dedup(np.array(a, dtype=np.int64))[0].tolist() == b


def test_spec_all_to_all_example():
    g = GOLD["all_to_all"]
    assert R.all_to_all(g["payloads"]) == g["expect"]
    with pytest.raises(ValueError):
        R.all_to_all([[1], [2, 3]])


def test_spec_stage_key_routing_example():
    g = GOLD["stage_key_routing"]
    batches = [(np.array(k, dtype=np.int64), np.array([0, len(k)], np.int32)) for k in g["worker_keys"]]
    _, own = R.route_all(batches, g["W"])
    assert [o.owner_keys.tolist() for o in own] == g["owner_requests"]


def _brute_route(keys, W, mb_occ, N):
    keys = [int(k) for k in keys]
    uniq = sorted(set(keys), key=lambda k: ((k & R.ROW_MASK) % W, k))
    inverse = [uniq.index(k) for k in keys]
    counts = [sum(1 for k in uniq if (k & R.ROW_MASK) % W == o) for o in range(W)]
    mask = [0] * len(uniq)
    for j, k in enumerate(keys):
        mask[uniq.index(k)] |= 1 << int(mb_occ[j])
    return uniq, inverse, counts, mask


@pytest.mark.parametrize("W,N,seed", [(1, 1, 0), (2, 2, 1), (3, 4, 2), (4, 3, 3)])
def test_route_source_brute_force(W, N, seed):
    cfg = WL.CONFIGS["tiny"]
    keys, offs = WL.gen_batch(cfg, seed, 0, 0, batch=24)
    perm, mbo = C.cluster_sequential(24, N) if 24 % N == 0 else C.cluster_sequential(24, 1)
    Nn = len(mbo) - 1
    mb = R.mb_of_occurrence(offs, cfg.num_features, perm, mbo)
    rs = R.route_source(keys, W, mb, Nn)
    uniq, inverse, counts, mask = _brute_route(keys, W, mb, Nn)
    assert rs.uniq.tolist() == uniq
    assert rs.inverse.tolist() == inverse
    assert rs.send_counts.tolist() == counts
    assert rs.send_offsets.tolist() == [0] + list(np.cumsum(counts))
    assert rs.mask.tolist() == mask
    # invariants named by BASELINE north_star: counts sum to unique keys and
    # every key lands on owner = row mod W
    assert rs.send_counts.sum() == len(set(keys.tolist()))
    for o in range(W):
        seg = rs.uniq[rs.send_offsets[o]:rs.send_offsets[o + 1]]
        assert ((seg & R.ROW_MASK) % W == o).all()
        assert (np.diff(seg) > 0).all()
    assert np.array_equal(rs.uniq[rs.inverse], keys)
    for i in range(Nn):
        has = [(m >> i) & 1 for m in mask]
        # pos_i = rank among mask-bit-i keys (brute force)
        for u in range(len(uniq)):
            if has[u]:
                assert rs.pos[i][u] == sum(has[:u])
        assert rs.mb_counts[i].sum() == sum(has)


def test_route_owner_conservation_and_dedup():
    cfg = WL.CONFIGS["tiny"]
    W, N = 3, 2
    batches = [WL.gen_batch(cfg, 7, 0, r, batch=16) for r in range(W)]
    mbs = [R.mb_of_occurrence(b[1], 4, *C.cluster_sequential(16, N)) for b in batches]
    src, own = R.route_all(batches, W, mbs, N)
    assert sum(s.send_counts.sum() for s in src) == sum(len(o.recv_keys) for o in own)
    for o, ow in enumerate(own):
        union = set()
        for s in range(W):
            union |= set(src[s].uniq[src[s].send_offsets[o]:src[s].send_offsets[o + 1]].tolist())
        assert ow.owner_keys.tolist() == sorted(union)              # P:347 second dedup
        assert np.array_equal(ow.owner_keys[ow.owner_inv], ow.recv_keys)
        for i in range(N):
            for s in range(W):
                lst = ow.send_lists[i][s]
                expect = [k for k in src[s].uniq[src[s].send_offsets[o]:src[s].send_offsets[o + 1]]
                          if (src[s].mask[np.searchsorted(src[s].uniq[src[s].send_offsets[o]:src[s].send_offsets[o+1]], k) + src[s].send_offsets[o]] >> i) & 1]
                assert ow.recv_keys[lst].tolist() == [int(k) for k in expect]


def test_microbatch_routing_resends():
    """keys repeated across micro-batches are re-sent; sum_i |K(M_i)| >= |K(B)|."""
    keys = np.array([5, 1, 5, 2], dtype=np.int64)
    offs = np.array([0, 2, 4], dtype=np.int32)          # sample0 {5,1}, sample1 {5,2}
    mb = R.mb_of_occurrence(offs, 1, np.array([0, 1]), np.array([0, 1, 2]))
    rs = R.route_source(keys, 1, mb, 2)
    assert rs.mb_counts[:, 0].tolist() == [2, 2]
    assert rs.mb_counts.sum() >= len(rs.uniq)


# ----------------------------------------------------------------------------- step
def test_spec_pool_examples():
    for c in GOLD["pool"]["cases"]:
        rows = np.array(c["rows"], dtype=np.float32)
        out = S.pool_sum(rows, np.array([0, len(rows)]))
        assert out[0].tolist() == c["expect"]
    # empty bag -> zero vector (reading Q5)
    assert S.pool_sum(np.zeros((0, 3), np.float32), np.array([0, 0])).tolist() == [[0, 0, 0]]


def test_spec_apply_sparse_grads_examples():
    c0, c1 = GOLD["apply_sparse_grads"]["cases"]
    out = S.sgd_rows(np.array([c0["e"]], np.float32), np.array([c0["sum"]]),
                     np.float32(c0["eta"] / c0["B"]))
    assert np.allclose(out[0], c0["expect"], rtol=1e-6)
    g = np.sum(np.array(c1["contribs"], dtype=np.float64), axis=0)
    out = S.sgd_rows(np.array([c1["e"]], np.float32), g[None], c1["eta"] / c1["B"])
    assert out[0].tolist() == c1["expect"]


def _brute_step(batches, douts, seed, d, mode, lr):
    """Plain per-key loops over the global batch (tiny inputs only)."""
    table = {}

    def get(k):
        if k not in table:
            table[k] = prf.init_rows(seed, np.array([k]), d, mode)[0].astype(np.float64)
        return table[k]
    pooled_all, grads = [], {}
    for (keys, offs), dout in zip(batches, douts):
        pooled = []
        for b in range(len(offs) - 1):
            acc = np.zeros(d)
            for j in range(offs[b], offs[b + 1]):
                acc = acc + get(int(keys[j]))
            pooled.append(acc.astype(np.float32))
            for j in range(offs[b], offs[b + 1]):
                k = int(keys[j])
                grads[k] = grads.get(k, np.zeros(d)) + dout[b].astype(np.float64)
        pooled_all.append(np.array(pooled))
    s = float(np.float32(lr))
    new = {k: (get(k) - s * g).astype(np.float32) for k, g in grads.items()}
    return pooled_all, new


@pytest.mark.parametrize("mode", ["dyadic", "uniform"])
def test_sync_step_brute_force(mode):
    cfg = WL.CONFIGS["tiny"]
    batches = [WL.gen_batch(cfg, 11, 0, r, batch=8) for r in range(2)]
    douts = [WL.gen_dout(11, 0, r, 8 * 4, 16, "dyadic" if mode == "dyadic" else "realistic")
             for r in range(2)]
    tab = S.LazyTable(4, 16, mode)
    res = S.sync_step(tab, batches, douts, 2.0 ** -10)
    pooled_bf, new_bf = _brute_step(batches, douts, 4, 16, mode, 2.0 ** -10)
    for a, b in zip(res.pooled, pooled_bf):
        if mode == "dyadic":
            assert np.array_equal(a, b)
        else:
            assert np.allclose(a, b, rtol=1e-6, atol=1e-7)
    for k, row in new_bf.items():
        got = tab.get(np.array([k]))[0]
        if mode == "dyadic":
            assert np.array_equal(got, row)
        else:
            assert np.allclose(got, row, rtol=1e-6, atol=1e-7)


def test_sync_step_closed_forms():
    # dpooled == 1 => G[k] = number of occurrences (exact, order free)
    cfg = WL.CONFIGS["tiny"]
    batches = [WL.gen_batch(cfg, 3, 0, r, batch=16) for r in range(2)]
    douts = [np.ones((16 * 4, 5), np.float32) for _ in range(2)]
    g = S.key_grads(batches, douts)
    allk = np.concatenate([b[0] for b in batches])
    for k, row, c in zip(g.keys, g.grad, g.count):
        n = int((allk == k).sum())
        assert c == n and (row == n).all()
    # constant rows c => pooled = bag length * c
    rows = np.full((int(batches[0][1][-1]), 5), 0.25, np.float32)
    pooled = S.pool_sum(rows, batches[0][1])
    assert np.array_equal(pooled[:, 0], np.diff(batches[0][1]) * 0.25)


def test_sync_step_only_touched_keys_change():
    """Eq. 2 first case: e_k unchanged for k not in K(B_t)."""
    cfg = WL.CONFIGS["tiny"]
    tab = S.LazyTable(0, 16)
    probe = np.array([(3 << 40) | 999, (0 << 40) | 998], dtype=np.int64)
    before = tab.get(probe).copy()
    batches = [WL.gen_batch(cfg, 0, 0, 0, batch=8)]
    assert not np.isin(probe, batches[0][0]).any()
    S.sync_step(tab, batches, [WL.gen_dout(0, 0, 0, 32, 16)], 0.5)
    assert np.array_equal(tab.get(probe), before)


def test_unpooled_forward_and_grads_hand_worked():
    """Unpooled variant (reading Q5, S:383-391 with one "bag" per occurrence):
    forward copies E_t[key_j] for every occurrence j in order; the gradient of
    key k is the sum of the dout rows of k's own occurrences, over the global
    batch (rank 0's occurrences before rank 1's).  Worked by hand:
    rank 0 keys [5, 7, 5, 9], rank 1 keys [7, 5]; dout row j (global index) = j + 1
    -> G[5] = 1 + 3 + 6 = 10, G[7] = 2 + 5 = 7, G[9] = 4; counts 3, 2, 1."""
    d = 4
    k0 = np.array([5, 7, 5, 9], np.int64)
    k1 = np.array([7, 5], np.int64)
    douts = [np.repeat(np.arange(1, 5, dtype=np.float32)[:, None], d, 1),
             np.repeat(np.arange(5, 7, dtype=np.float32)[:, None], d, 1)]
    batches = [(k0, np.arange(5)), (k1, np.arange(3))]
    g = S.key_grads(batches, douts, pooling="none")
    assert g.keys.tolist() == [5, 7, 9]
    assert g.grad[:, 0].tolist() == [10.0, 7.0, 4.0] and (g.grad == g.grad[:, :1]).all()
    assert g.count.tolist() == [3, 2, 1]
    # a pooled batch with the SAME keys in bags would give key 5 the bag
    # gradients instead: [5,7] [5,9] bags with dout 1, 2 -> G[5] = 3 (differs)
    gp = S.key_grads([(k0, np.array([0, 2, 4]))], [np.array([[1.0] * d, [2.0] * d], np.float32)])
    assert gp.grad[0, 0] == 3.0
    tab = S.LazyTable(2, d, "dyadic")
    out = S.forward(tab, k0, np.arange(5), pooling="none")
    assert out.shape == (4, d)
    assert np.array_equal(out, prf.init_rows(2, k0, d, "dyadic"))   # row per occurrence, in order
    assert np.array_equal(out[0], out[2])                           # repeated key -> same row
    # the step: e' = e - s G, exact in the dyadic regime
    before = prf.init_rows(2, np.array([5, 7, 9], np.int64), d, "dyadic").astype(np.float64)
    res = S.sync_step(tab, batches, douts, 2.0 ** -4, pooling="none")
    assert np.array_equal(res.pooled[1], prf.init_rows(2, k1, d, "dyadic"))
    want = (before - 2.0 ** -4 * np.array([[10.0], [7.0], [4.0]])).astype(np.float32)
    assert np.array_equal(tab.get(np.array([5, 7, 9])), want)


def test_unpooled_equals_pooled_for_single_key_bags():
    """Special case: when every bag holds exactly one key, sum pooling is the
    identity, so the pooled and unpooled steps coincide (forward and grads)."""
    cfg = WL.CONFIGS["tiny"].with_(bag_len=(1, 1))
    batches = [WL.gen_batch(cfg, 5, 0, r, batch=8) for r in range(2)]
    assert all((np.diff(o) == 1).all() for _, o in batches)
    douts = [WL.gen_dout(5, 0, r, 8 * 4, 16, "realistic") for r in range(2)]
    gs, gn = S.key_grads(batches, douts, "sum"), S.key_grads(batches, douts, "none")
    assert np.array_equal(gs.keys, gn.keys) and np.array_equal(gs.grad, gn.grad)
    tab = S.LazyTable(1, 16)
    for k, o in batches:
        assert np.array_equal(S.forward(tab, k, o, "sum"), S.forward(tab, k, o, "none"))


# ----------------------------------------------------------------------------- cluster
def test_spec_cluster_example():
    g = GOLD["cluster_samples"]
    ks = [np.array(k) for k in g["keysets"]]
    for fn in (C.cluster_rounds, C.cluster_spec_greedy):
        perm, mbo = fn(ks, g["N"])
        groups = [sorted(perm[mbo[i]:mbo[i + 1]].tolist()) for i in range(g["N"])]
        assert sorted(groups) == g["groups"]
        assert C.partition_cost(ks, perm, mbo) == g["cost"]
    assert C.brute_force_best(ks, 2) == g["cost"]
    assert C.partition_cost(ks, np.array([0, 2, 1, 3]), np.array([0, 2, 4])) == g["random_pair_cost"]


def test_cluster_n1_and_ties_and_validity():
    ks = [np.array([1, 2])] * 6
    for fn in (C.cluster_rounds, C.cluster_spec_greedy):
        perm, mbo = fn(ks, 1)
        assert perm.tolist() == list(range(6))
        perm, mbo = fn(ks, 3)
        # identical sets: deterministic, lowest-id tie break
        assert np.array_equal(perm, fn(ks, 3)[0])
        assert sorted(perm.tolist()) == list(range(6))
    with pytest.raises(ValueError):
        C.cluster_rounds(ks, 4)


def test_admission_schedule():
    g = C.admission_sizes(10 ** 9)
    assert [next(g) for _ in range(7)] == [1, 1, 1, 2, 3, 3, 4]


# the hand-worked multi-round example of test_cluster_rounds_hand_worked
HAND_KEYSETS = [
    {1, 2, 3, 4}, {10, 11, 12, 13}, {1, 2, 5}, {1, 2}, {10, 11, 14}, {10, 11, 15},
    {3, 4, 5, 6}, {12, 13, 16}, {5, 6, 7}, {1, 16, 17}, {7, 8}, {18, 19},
]
HAND_PERM = [0, 2, 3, 6, 8, 9, 1, 4, 5, 7, 10, 11]


def test_cluster_rounds_hand_worked():
    """SURVEY §8(c) "Clustering spec", worked by hand on B = 12, N = 2
    (cap = 6), so that rounds 1-3 admit q = 1 and round 4 admits q = 2
    (schedule 1, 1, 1, 2).  S = overlap with the group's union, growth = size - S.

    Seeds.  g0: largest sample; sizes 4 = {id0, id1, id6} -> lowest id: id0,
    U0 = {1,2,3,4}.  g1: min overlap with U0, then size desc: overlap 0 and
    size 4 only id1 -> U1 = {10,11,12,13}.
    Round 1 (q = 1), snapshot U0 = {1..4}, U1 = {10..13}:
      g0: S = 2 for id2 (growth 1), id3 (growth 0), id6 (growth 2)
          -> id3  [S tie broken by growth asc]
      g1: S = 2, growth 1 for id4, id5, id7 -> id4  [S and growth tie broken by id]
      unions after the round: U0 = {1..4}, U1 = {10..14}.
    Round 2 (q = 1): g0: S = 2 for id2 (growth 1), id6 (growth 2) -> id2;
      g1: S = 2, growth 1 for id5, id7 -> id5.  U0 = {1..5}, U1 = {10..15}.
    Round 3 (q = 1): g0: id6 S = 3 (others <= 1) -> id6;
      g1: id7 S = 2 (others 0) -> id7.  U0 = {1..6}, U1 = {10..16}.
    Round 4 (q = 2, have 4 each): snapshot S0: id8 {5,6,7} 2; id9 {1,16,17} 1;
      id10 {7,8} 0 (growth 2); id11 {18,19} 0 (growth 2) -> g0 takes id8, id9;
      g1 takes the rest, id10, id11.
    Result: g0 = {0,2,3,6,8,9}, g1 = {1,4,5,7,10,11}.

    Plausible misreadings give other partitions (checked below):
      * the union growing inside a round (g0 re-ranks after id8: id10 {7,8}
        then has S 1 / growth 1 and beats id9) -> g0 gets id10;
      * admission size fixed at 1 (round 4: g0 takes id8, g1 takes id9, whose
        key 16 is in U1);
      * growth tie broken desc (round 1: g0 takes id6); id tie broken desc
        (round 1: g1 takes id7); seed ties to the highest id (seed id6).
    """
    ks = [np.array(sorted(k), dtype=np.int64) for k in HAND_KEYSETS]
    perm, mbo = C.cluster_rounds(ks, 2)
    assert perm.tolist() == HAND_PERM
    assert mbo.tolist() == [0, 6, 12]
    mb = C.mb_of_sample(perm, mbo, 12)
    # the misreadings above assign these samples differently
    assert mb[9] == 0 and mb[10] == 1 and mb[3] == 0 and mb[6] == 0 and mb[4] == 1 and mb[7] == 1
    assert C.partition_cost(ks, perm, mbo) == 9 + 11


@pytest.mark.parametrize("seed", range(4))
def test_cluster_rounds_valid_partitions(seed):
    """Partition validity: disjoint, equal-sized groups covering the batch."""
    rng = np.random.default_rng(seed)
    ks = [np.unique(rng.integers(0, 8, size=rng.integers(1, 4))) for _ in range(6)]
    for N in (1, 2, 3):
        perm, mbo = C.cluster_rounds(ks, N)
        assert sorted(perm.tolist()) == list(range(6))
        assert mbo.tolist() == [i * (6 // N) for i in range(N + 1)]
        # within a group, samples are listed by ascending id (perm = sort by (group, id))
        for i in range(N):
            g = perm[mbo[i]:mbo[i + 1]].tolist()
            assert g == sorted(g)


def test_cluster_payload_dominance_correlated():
    """S:586 / A6: mean clustered sum_i |K(M_i)| <= mean random."""
    cfg = WL.CONFIGS["tiny"].with_(table_rows=(2000,) * 4)
    tot_c = tot_r = 0
    for seed in range(6):
        keys, offs = WL.gen_correlated_batch(cfg, seed, 0, 0, groups=8, rho=0.8, batch=64)
        ks = C.sample_keysets(keys, offs, 4)
        tot_c += C.partition_cost(ks, *C.cluster_rounds(ks, 4))
        rp = np.random.default_rng(seed).permutation(64)
        tot_r += C.partition_cost(ks, rp, np.arange(5) * 16)
    assert tot_c < tot_r


# ----------------------------------------------------------------------------- pipeline
def test_spec_dual_buffer_sync_example():
    g = GOLD["dual_buffer_sync"]
    mk = lambda d: P.Buffer(0, np.array(sorted(int(k) for k in d)),
                            np.array([d[str(k)] for k in sorted(int(k) for k in d)], np.float32))
    a, p = mk(g["active"]), mk(g["prefetch"])
    P.dual_buffer_sync(a, p)
    assert {int(k): r.tolist() for k, r in zip(p.keys, p.rows)} == \
        {int(k): np.float32(v).tolist() for k, v in g["expect"].items()}
    # disjoint -> unchanged; identical -> copy
    q = mk({"9": [4.0]})
    P.dual_buffer_sync(a, q)
    assert q.rows.tolist() == [[4.0]]
    r = mk({"5": [0.0], "7": [0.0]})
    P.dual_buffer_sync(a, r)
    assert np.array_equal(r.rows, a.rows)


def _tiny_traj(W, T=6, seed=0, batch=8, dyadic=True):
    cfg = WL.CONFIGS["tiny"]
    batches = [[WL.gen_batch(cfg, seed, t, r, batch=batch) for r in range(W)] for t in range(T)]
    douts = [[WL.gen_dout(seed, t, r, batch * 4, 16, "dyadic" if dyadic else "realistic")
              for r in range(W)] for t in range(T)]
    return batches, douts


@pytest.mark.parametrize("W,N,cl,grad", [(1, 1, "sequential", "lin"), (2, 2, "clustered", "lin"),
                                         (4, 4, "clustered", "quad"), (2, 4, "sequential", "quad"),
                                         (3, 2, "clustered", "lin")])
def test_corollary1_pipelined_equals_sync_bitwise(W, N, cl, grad):
    """Corollary 1 in parity regime P1: DBP+FWP tables == Eq. 1."""
    batches, douts = _tiny_traj(W)
    lr = 2.0 ** -10
    ref = P.sync_train(S.LazyTable(1, 16, "dyadic"), batches, douts, lr, grad_mode=grad)
    tr = P.nestpipe_train(S.LazyTable(1, 16, "dyadic"), batches, douts,
                          P.PipeConfig(W=W, N=N, cluster=cl, F=4, lr_over_B=lr, grad_mode=grad))
    assert P.first_divergence(ref, [t.table for t in tr]) is None
    # forward rows: pooled of every micro-batch equals the sync forward
    tab = S.LazyTable(1, 16, "dyadic")
    res = S.sync_step(tab, batches[0], douts[0], lr, grad_mode=grad)
    for r in range(W):
        for i in range(N):
            perm, mbo = tr[0].perm[r], tr[0].mb_offsets[r]
            bags = P._mb_bags(perm, mbo, i, 4)
            assert np.array_equal(tr[0].pooled[r][i], res.pooled[r][bags])


def test_negative_control_six_stage_diverges_at_step2():
    """P:436-440 / S:473, S:732 (A3): skipping the dual-buffer sync gives a
    one-step-stale read; divergence first appears at step 2 (1-based)."""
    W = 2
    cfg = WL.CONFIGS["tiny"]
    hot = np.int64(7)
    batches, douts = _tiny_traj(W)
    # adversarial: one hot key in every batch of every rank
    batches = [[(np.concatenate([[hot], k[1:]]), o) for (k, o) in st] for st in batches]
    lr = 2.0 ** -6
    ref = P.sync_train(S.LazyTable(1, 16, "dyadic"), batches, douts, lr, grad_mode="quad")
    safe = P.nestpipe_train(S.LazyTable(1, 16, "dyadic"), batches, douts,
                            P.PipeConfig(W=W, N=2, F=4, lr_over_B=lr, grad_mode="quad"))
    bad = P.nestpipe_train(S.LazyTable(1, 16, "dyadic"), batches, douts,
                           P.PipeConfig(W=W, N=2, F=4, lr_over_B=lr, grad_mode="quad",
                                        unsafe_six_stage=True))
    assert P.first_divergence(ref, [t.table for t in safe]) is None
    assert P.first_divergence(ref, [t.table for t in bad], tol=1e-6) == 2
    # tau = 1: the stale row the unsafe run used at step 2 is the oracle's step-0 init value
    rows0 = S.LazyTable(1, 16, "dyadic").get(np.array([hot]))[0]
    assert not np.array_equal(ref[0][int(hot)], rows0)


def test_pipeline_depth_and_n_independence():
    """S:496 depth independence + Prop. 2: N and clustering do not
    change the tables (P1, bitwise)."""
    batches, douts = _tiny_traj(2)
    runs = []
    for pipelined, N, cl in [(False, 1, "sequential"), (True, 1, "sequential"),
                             (True, 2, "clustered"), (True, 4, "sequential")]:
        tr = P.nestpipe_train(S.LazyTable(2, 16, "dyadic"), batches, douts,
                              P.PipeConfig(W=2, N=N, cluster=cl, F=4, pipelined=pipelined))
        runs.append([t.table for t in tr])
    for r in runs[1:]:
        assert P.first_divergence(runs[0], r) is None


def test_realistic_regime_pipelined_close_to_sync():
    batches, douts = _tiny_traj(2, dyadic=False)
    ref = P.sync_train(S.LazyTable(1, 16), batches, douts, 0.05)
    tr = P.nestpipe_train(S.LazyTable(1, 16), batches, douts,
                          P.PipeConfig(W=2, N=2, cluster="clustered", F=4, lr_over_B=0.05))
    assert P.first_divergence(ref, [t.table for t in tr], tol=1e-6) is None


# ----------------------------------------------------------------------------- workload
def test_workload_deterministic_and_skewed():
    cfg = WL.CONFIGS["tiny"]
    a = WL.gen_batch(cfg, 1, 2, 0)
    b = WL.gen_batch(cfg, 1, 2, 0)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    keys, offs = a
    assert len(offs) == 32 * 4 + 1 and (np.diff(offs) >= 1).all() and (np.diff(offs) <= 3).all()
    tab, row = WL.unpack_keys(keys)
    F = 4
    bag_tab = np.repeat(np.arange(32 * F) % F, np.diff(offs))
    assert np.array_equal(tab, bag_tab) and (row < 1000).all()
    # no repeats within a bag
    for bg in range(32 * F):
        seg = keys[offs[bg]:offs[bg + 1]]
        assert len(np.unique(seg)) == len(seg)
    r = WL.zipf_ranks(np.random.default_rng(0), 1.2, 10 ** 4, 10 ** 5)
    cnt = np.bincount(r, minlength=10 ** 4)
    assert cnt[0] > cnt[99] > 0


# --------------------------------------------------------------------------- row-wise AdaGrad (NEXT-2)
def _one_bag_step(opt, dout_rows, keys_per_bag, seed=3, d=4):
    """One sync step: bag b holds keys_per_bag[b] (one rank), dpooled = dout_rows."""
    keys = np.array([k for ks in keys_per_bag for k in ks], np.int64)
    offs = np.concatenate([[0], np.cumsum([len(ks) for ks in keys_per_bag])]).astype(np.int64)
    tab = S.LazyTable(seed, d, "dyadic")
    before = {int(k): tab.get([k])[0].copy() for k in np.unique(keys)}
    S.sync_step(tab, [(keys, offs)], [np.asarray(dout_rows, np.float32)], 0.0, optimizer=opt)
    return tab, before


def test_adagrad_first_steps_closed_form():
    """eps = 0, uniform gradient c: step 1 moves every element by exactly
    -lr*sign(c) (m = c^2); step 2 by -lr*sign(c)/sqrt(2) (m = 2c^2)."""
    k, c, lr = (2 << 40) | 17, -2.0 ** -3, 2.0 ** -4
    opt = S.RowwiseAdagrad(lr=lr, grad_scale=1.0, eps=0.0)
    tab, before = _one_bag_step(opt, [[c] * 4], [[k]])
    e1 = tab.get([k])[0]
    assert np.array_equal(e1, (before[k].astype(np.float64) + lr).astype(np.float32))
    assert opt.get_state([k])[0] == c * c
    keys, offs = np.array([k], np.int64), np.array([0, 1], np.int64)
    S.sync_step(tab, [(keys, offs)], [np.full((1, 4), c, np.float32)], 0.0, optimizer=opt)
    e2 = tab.get([k])[0]
    assert np.array_equal(e2, (e1.astype(np.float64) + lr / np.sqrt(2.0)).astype(np.float32))
    assert opt.get_state([k])[0] == 2 * c * c


def test_adagrad_rowwise_mean_and_sum_before_square():
    """m is the mean over d of the squared SUMMED gradient: g = (3,4,0,0)/16
    gives sqrt(m) = 2.5/16, so the step is lr*(1.2, 1.6, 0, 0); a key in two
    bags with gradient c each moves like one bag with 2c (sum, then square)."""
    k, lr = (1 << 40) | 5, 2.0 ** -3
    opt = S.RowwiseAdagrad(lr=lr, grad_scale=1.0, eps=0.0)
    tab, before = _one_bag_step(opt, [[3 / 16, 4 / 16, 0, 0]], [[k]])
    want = (before[k].astype(np.float64) - lr * np.array([1.2, 1.6, 0.0, 0.0])).astype(np.float32)
    assert np.allclose(tab.get([k])[0], want, rtol=0, atol=1e-7)
    c = 2.0 ** -5
    opt2 = S.RowwiseAdagrad(lr=lr, grad_scale=1.0, eps=0.0)
    tab2, before2 = _one_bag_step(opt2, [[c] * 4, [c] * 4], [[k], [k]])
    assert np.array_equal(tab2.get([k])[0], (before2[k].astype(np.float64) - lr).astype(np.float32))
    assert opt2.get_state([k])[0] == (2 * c) ** 2


def test_adagrad_grad_scale_eps_and_untouched_keys():
    """grad_scale scales g before squaring; eps enters the denominator; keys
    outside K(B_t) keep their rows and accumulators."""
    k, other, lr, gs, eps = (0 << 40) | 9, (0 << 40) | 10, 2.0 ** -2, 2.0 ** -2, 2.0 ** -4
    opt = S.RowwiseAdagrad(lr=lr, grad_scale=gs, eps=eps, init=2.0 ** -6)
    tab, before = _one_bag_step(opt, [[1.0] * 4], [[k]])
    g = gs * 1.0
    m = 2.0 ** -6 + g * g
    want = (before[k].astype(np.float64) - lr * g / (np.sqrt(m) + eps)).astype(np.float32)
    assert np.array_equal(tab.get([k])[0], want)
    assert opt.get_state([other])[0] == 2.0 ** -6
    assert np.array_equal(tab.get([other])[0], S.LazyTable(3, 4, "dyadic").get([other])[0])


@pytest.mark.parametrize("W,N,cl", [(2, 1, "sequential"), (2, 2, "clustered"), (3, 2, "sequential")])
def test_adagrad_pipelined_equals_sync_bitwise(W, N, cl):
    """Corollary 1 with row-wise AdaGrad: the accumulator lives with the
    owner's row and is read and written only by the update, so DBP+FWP still
    reproduce the synchronous step bit for bit (P1 gradients)."""
    batches, douts = _tiny_traj(W)
    mk = lambda: S.RowwiseAdagrad(lr=2.0 ** -6, grad_scale=2.0 ** -5, eps=1e-8)
    ref = P.sync_train(S.LazyTable(1, 16, "dyadic"), batches, douts, 0.0, optimizer=mk())
    tr = P.nestpipe_train(S.LazyTable(1, 16, "dyadic"), batches, douts,
                          P.PipeConfig(W=W, N=N, cluster=cl, F=4, optimizer=mk()))
    assert P.first_divergence(ref, [t.table for t in tr]) is None
