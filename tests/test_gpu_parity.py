"""GPU parity: libnest.so (through the C ABI) vs the CPU oracle (-m gpu).

Bar (BASELINE north_star): keys, routing, counts and offsets bit-exact;
pooled rows, gradients and tables within 1e-5 relative (normwise per row,
SURVEY §8(c) Q13) -- and bit-exact in parity regime P1 (dyadic values, where
every sum is exact in fp32).
"""
import numpy as np
import pytest

import workload as WL
from oracle import cluster as OC
from oracle import pipeline as OP
from oracle import prf as OPRF
from oracle import routing as OR
from oracle import step as OS

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2604_06956_b200 import NestContext, NestError  # noqa: E402
from paper_2604_06956_b200.runner import Runner  # noqa: E402

DEV = torch.device("cuda:0")


def to_dev(a, dtype):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV, dtype)


def make_ctx(cfg, B, N=1, K=None, init="dyadic", seed=1, **kw):
    K = K or int(B * cfg.num_features * cfg.bag_len[1])
    return NestContext(cfg.table_rows, cfg.dim, pooling=cfg.pooling, num_features=cfg.num_features, max_keys=K,
                       max_batch=B, max_micro_batches=N, seed=seed, init_mode=init, device=DEV, **kw)


def rel_rowwise_ok(gpu, ref, tol=1e-5, scale=None):
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    num = np.linalg.norm(gpu - ref, axis=1)
    den = np.linalg.norm(ref if scale is None else scale, axis=1)
    return np.all(num <= tol * np.maximum(den, 1e-30))


# --------------------------------------------------------------------------- init
@pytest.mark.parametrize("init", ["uniform", "dyadic"])
def test_init_tables_match_prf(init):
    cfg = WL.CONFIGS["tiny"]
    ctx = make_ctx(cfg, 32, init=init, seed=7)
    keys = np.array([(t << 40) | r for t in range(4) for r in (0, 1, 17, 500, 999)], dtype=np.int64)
    got = ctx.read_rows(to_dev(keys, torch.int64)).cpu().numpy()
    ref = OPRF.init_rows(7, keys, cfg.dim, init)
    assert np.array_equal(got, ref)


# --------------------------------------------------------------------------- route
@pytest.mark.parametrize("N,B,seed", [(1, 32, 0), (2, 32, 1), (4, 64, 2), (8, 64, 3)])
def test_route_w1_bit_exact(N, B, seed):
    cfg = WL.CONFIGS["tiny"]
    keys, offs = WL.gen_batch(cfg, seed, 0, 0, batch=B)
    ctx = make_ctx(cfg, B, N=N)
    perm, mbo = ctx.fwp_schedule(None, None, B, N, "sequential")
    ctx.route(0, to_dev(keys, torch.int64), to_dev(offs, torch.int32), B, perm=perm, mb_offsets=mbo, N=N)
    v = ctx.route_view(0)
    mb = OR.mb_of_occurrence(offs, cfg.num_features, perm.cpu().numpy(), mbo.cpu().numpy())
    rs = OR.route_source(keys, 1, mb, N)
    assert np.array_equal(v["uniq"], rs.uniq)
    assert np.array_equal(v["inverse"], rs.inverse)
    assert np.array_equal(v["mask"].astype(np.int64), rs.mask)
    assert np.array_equal(v["pos"].astype(np.int64), rs.pos)
    assert v["send_counts"][0, 0] == rs.send_counts[0]
    assert np.array_equal(v["send_counts"][0, 1:1 + N], rs.mb_counts[:, 0])
    # owner side at W=1: owner rows are the shard rows of uniq, ascending
    assert v["n_owner"] == len(rs.uniq)
    tab, row = WL.unpack_keys(rs.uniq)
    assert np.array_equal(v["owner_rows"], tab * 1000 + row)
    # the gathered buffer equals the PRF rows of uniq (R4)
    assert np.array_equal(v["buffer"], OPRF.init_rows(1, rs.uniq, cfg.dim, "dyadic"))


def test_route_mid_size_radix_tiles_and_ragged_tail():
    """Several radix tiles (4096) with a ragged tail, heavy skew -> hot keys."""
    cfg = WL.CONFIGS["tiny"].with_(table_rows=(5000, 3000, 200, 77), zipf=1.3, bag_repeats=True)
    B = 3000
    keys, offs = WL.gen_batch(cfg, 5, 0, 0, batch=B)
    ctx = make_ctx(cfg, B, N=4, K=len(keys) + 11)
    perm, mbo = ctx.fwp_schedule(None, None, B, 4, "sequential")
    ctx.route(1, to_dev(keys, torch.int64), to_dev(offs, torch.int32), B, perm=perm, mb_offsets=mbo, N=4)
    v = ctx.route_view(1)
    mb = OR.mb_of_occurrence(offs, 4, perm.cpu().numpy(), mbo.cpu().numpy())
    rs = OR.route_source(keys, 1, mb, 4)
    assert np.array_equal(v["uniq"], rs.uniq)
    assert np.array_equal(v["inverse"], rs.inverse)
    assert np.array_equal(v["mask"].astype(np.int64), rs.mask)
    assert np.array_equal(v["pos"].astype(np.int64), rs.pos)


# --------------------------------------------------------------------------- row-wise AdaGrad
@pytest.mark.parametrize("N,pipelined", [(1, True), (2, True), (1, False)])
def test_train_w1_rowwise_adagrad_vs_oracle(N, pipelined):
    """NEXT-2: the update with row-wise AdaGrad (tables and accumulators after
    T steps) against oracle.step.RowwiseAdagrad, 1e-5 row-wise (P2)."""
    cfg = WL.CONFIGS["tiny"].with_(table_rows=(5000, 3000, 200, 77), zipf=1.3, bag_repeats=True, dim=32)
    B, T, F, d, seed = 256, 5, cfg.num_features, cfg.dim, 7
    batches = [[WL.gen_batch(cfg, seed, t, 0, batch=B)] for t in range(T)]
    douts = [[WL.gen_dout(seed, t, 0, B * F, d, "realistic")] for t in range(T)]
    K = max(len(b[0][0]) for b in batches)
    gs, lr, eps = 1.0 / B, 0.05, 1e-8
    ctx = make_ctx(cfg, B, N=N, K=K, init="uniform", seed=11, optimizer="rowwise_adagrad", adagrad_eps=eps)
    run = Runner(ctx, N=N, pipelined=pipelined, adagrad=(gs, lr))
    dev_b = [(to_dev(b[0][0], torch.int64), to_dev(b[0][1], torch.int32), B) for b in batches]
    cap = B // N
    # every step's dout stays referenced until the end: the library reads it
    # asynchronously on its own streams (the caller owns input lifetimes)
    dds = [to_dev(douts[t][0], torch.float32) for t in range(T)]
    for t in range(T):
        run.step(dev_b[t], dev_b[t + 1] if t + 1 < T else None,
                 lambda tt, i, p, dd=dds[t]: dd[i * cap * F:(i + 1) * cap * F])
    run.join()
    torch.cuda.synchronize()
    tab = OS.LazyTable(11, d, "uniform")
    opt = OS.RowwiseAdagrad(lr=lr, grad_scale=gs, eps=eps)
    for t in range(T):
        OS.sync_step(tab, batches[t], douts[t], 0.0, optimizer=opt)
    allk = np.unique(np.concatenate([b[0][0] for b in batches]))
    kd = to_dev(allk, torch.int64)
    assert rel_rowwise_ok(ctx.read_rows(kd).cpu().numpy(), tab.get(allk))
    m = ctx.read_state(kd).cpu().numpy().astype(np.float64)
    ref_m = opt.get_state(allk)
    assert np.all(np.abs(m - ref_m) <= 1e-5 * ref_m + 1e-30)
    assert (ref_m > 0).all()


def test_rowwise_adagrad_errors():
    cfg = WL.CONFIGS["tiny"]
    sgd = make_ctx(cfg, 32)
    with pytest.raises(NestError):
        sgd.read_state(to_dev(np.array([0], np.int64), torch.int64))
    ada = make_ctx(cfg, 32, optimizer="rowwise_adagrad")
    keys, offs = WL.gen_batch(cfg, 1, 0, 0, batch=32)
    ada.route(0, to_dev(keys, torch.int64), to_dev(offs, torch.int32), 32)
    out = torch.empty((32 * cfg.num_features, cfg.dim), dtype=torch.float32, device=DEV)
    ada.lookup_fwd(0, 0, out)
    with pytest.raises(NestError):
        ada.grad_bwd_update(0, 0, out, 0.1)          # SGD call on an AdaGrad context
    ada.grad_bwd_update_adagrad(0, 0, out, 1 / 32, 0.1)
    torch.cuda.synchronize()


# --------------------------------------------------------------------------- bf16 hand-off
def test_lookup_bf16_and_tower_bf16_input_match_fp32_path():
    """nest_lookup_fwd_bf16 == bf16(RN) of nest_lookup_fwd bit for bit, and the
    tower's input gradient from the bf16 rows == the one from the fp32 rows
    (cast inside) bit for bit; the fp32 rows meet the oracle's P2 bar."""
    cfg = WL.CONFIGS["tiny"].with_(table_rows=(5000, 3000, 200, 77), zipf=1.3, bag_repeats=True, dim=64)
    B = 512
    keys, offs = WL.gen_batch(cfg, 9, 0, 0, batch=B)
    ctx = make_ctx(cfg, B, K=len(keys), init="uniform", seed=4, tower_layers=2, tower_hidden=64)
    ctx.route(0, to_dev(keys, torch.int64), to_dev(offs, torch.int32), B)
    rows = B * cfg.num_features
    out32 = torch.empty((rows, cfg.dim), dtype=torch.float32, device=DEV)
    out16 = torch.empty((rows, cfg.dim), dtype=torch.bfloat16, device=DEV)
    ctx.lookup_fwd(0, 0, out32)
    ctx.lookup_fwd(0, 0, out16)
    torch.cuda.synchronize()
    assert torch.equal(out16.view(torch.int16), out32.to(torch.bfloat16).view(torch.int16))
    tab = OS.LazyTable(4, cfg.dim, "uniform")
    ref = OS.forward(tab, keys, offs, pooling="sum")
    assert rel_rowwise_ok(out32.cpu().numpy(), ref)
    d32 = torch.empty((rows, cfg.dim), dtype=torch.float32, device=DEV)
    d16 = torch.empty_like(d32)
    ctx.tower_fwd_bwd(out32, d32)
    ctx.tower_fwd_bwd(out16, d16)
    ctx.join()
    torch.cuda.synchronize()
    assert torch.isfinite(d32).all() and d32.abs().sum() > 0
    assert torch.equal(d32, d16)


# --------------------------------------------------------------------------- full steps
def _run_w1(cfg, B, N, T, init, dmode, lr, pipelined, seed=3, grad_mode="lin"):
    F, d = cfg.num_features, cfg.dim
    batches = [[WL.gen_batch(cfg, seed, t, 0, batch=B)] for t in range(T)]
    pooled_mode = cfg.pooling == "sum"
    douts = [[WL.gen_dout(seed, t, 0, B * F if pooled_mode else len(batches[t][0][0]), d, dmode)]
             for t in range(T)]
    K = max(len(b[0][0]) for b in batches)
    ctx = make_ctx(cfg, B, N=N, K=K, init=init, seed=11)
    run = Runner(ctx, N=N, pipelined=pipelined, lr_over_B=lr)
    dev_b = [(to_dev(b[0][0], torch.int64), to_dev(b[0][1], torch.int32), B) for b in batches]
    pooled_gpu = []
    for t in range(T):
        cap = B // N

        def dout_fn(tt, i, pooled, t=t):
            if grad_mode == "quad":
                return pooled
            if pooled_mode:
                return to_dev(douts[t][0][i * cap * F:(i + 1) * cap * F], torch.float32)
            o = batches[t][0][1]
            return to_dev(douts[t][0][o[i * cap * F]:o[(i + 1) * cap * F]], torch.float32)
        outs = run.step(dev_b[t], dev_b[t + 1] if t + 1 < T else None, dout_fn)
        torch.cuda.synchronize()
        pooled_gpu.append([o.cpu().numpy() for o in outs])
    tab = OS.LazyTable(11, d, init)
    ref_pooled, ref_rows = [], []
    for t in range(T):
        res = OS.sync_step(tab, batches[t], douts[t], lr, pooling=cfg.pooling, grad_mode=grad_mode)
        ref_pooled.append(res.pooled[0])
    allk = np.unique(np.concatenate([b[0][0] for b in batches]))
    got = ctx.read_rows(to_dev(allk, torch.int64)).cpu().numpy()
    return pooled_gpu, ref_pooled, got, tab.get(allk), tab


@pytest.mark.parametrize("N,pipelined,grad", [(1, False, "lin"), (1, True, "lin"), (2, True, "lin"),
                                              (4, True, "quad"), (8, False, "lin")])
def test_train_w1_dyadic_bit_exact(N, pipelined, grad):
    """P1: 10 steps, pooled rows of every step and the final tables bit-exact.
    QUAD couples dout to the pooled values, whose dyadic resolution halves
    with every update, so past step 2 it is compared in regime P2 (1e-5)."""
    cfg = WL.CONFIGS["tiny"]
    B = 32
    pg, pr, got, ref, _ = _run_w1(cfg, B, N, 10, "dyadic", "dyadic", 2.0 ** -10, pipelined, grad_mode=grad)
    for t in range(10):
        if grad == "lin" or t < 2:
            assert np.array_equal(np.concatenate(pg[t]), pr[t]), f"pooled step {t}"
        else:
            assert rel_rowwise_ok(np.concatenate(pg[t]), pr[t]), f"pooled step {t}"
    if grad == "lin":
        assert np.array_equal(got, ref)
    else:
        assert rel_rowwise_ok(got, ref)


def test_train_w1_realistic_within_tolerance():
    """P2: uniform init, normal gradients, 10 steps: 1e-5 relative per row."""
    cfg = WL.CONFIGS["tiny"]
    B = 64
    pg, pr, got, ref, _ = _run_w1(cfg, B, 4, 10, "uniform", "realistic", 0.05, True)
    for t in range(10):
        assert rel_rowwise_ok(np.concatenate(pg[t]), pr[t])
    assert rel_rowwise_ok(got, ref)


def test_train_mid_size_hot_segments_p1():
    """Hot keys with thousands of occurrences exercise the chunked two-level
    segment reduce; P1 keeps the comparison bit-exact."""
    cfg = WL.CONFIGS["tiny"].with_(table_rows=(4000, 50, 9, 2000), zipf=1.4, bag_repeats=True, dim=128)
    B = 4096
    pg, pr, got, ref, _ = _run_w1(cfg, B, 2, 3, "dyadic", "dyadic", 2.0 ** -12, True)
    for t in range(3):
        assert np.array_equal(np.concatenate(pg[t]), pr[t])
    assert np.array_equal(got, ref)


def test_run_to_run_bitwise_deterministic():
    cfg = WL.CONFIGS["tiny"].with_(zipf=1.3, bag_repeats=True)
    a = _run_w1(cfg, 256, 2, 3, "uniform", "realistic", 0.1, True)[2]
    b = _run_w1(cfg, 256, 2, 3, "uniform", "realistic", 0.1, True)[2]
    assert np.array_equal(a, b)


@pytest.mark.parametrize("d", [16, 32, 64, 256])
def test_dims(d):
    cfg = WL.CONFIGS["tiny"].with_(dim=d)
    pg, pr, got, ref, _ = _run_w1(cfg, 32, 2, 3, "dyadic", "dyadic", 2.0 ** -10, True)
    assert np.array_equal(got, ref)


def test_unpooled_expand_p1():
    cfg = WL.CONFIGS["tiny"].with_(pooling="none", bag_len=(4, 9), bag_repeats=True)
    B = 32
    pg, pr, got, ref, _ = _run_w1(cfg, B, 2, 3, "dyadic", "dyadic", 2.0 ** -10, True)
    for t in range(3):
        assert np.array_equal(np.concatenate(pg[t]), pr[t])
    assert np.array_equal(got, ref)


# --------------------------------------------------------------------------- clustering
@pytest.mark.parametrize("case", ["tiny-N2", "tiny-N4", "corr-N4", "corr-N8", "dlrmish-N4", "longbag-N4"])
def test_cluster_bit_exact_vs_oracle(case):
    """R14: GPU round-based greedy == oracle.cluster.cluster_rounds (perm + offsets).
    longbag: > 127 distinct keys per sample, so the rank keys need the second
    histogram level of the select."""
    if case.startswith("longbag"):
        cfg = WL.CONFIGS["tiny"].with_(table_rows=(20000,) * 4, bag_len=(30, 60), bag_repeats=True, zipf=1.1)
        B, N = 256, 4
        keys, offs = WL.gen_batch(cfg, 6, 0, 0, batch=B)
        assert max(len(k) for k in OC.sample_keysets(keys, offs, cfg.num_features)) > 127
    elif case.startswith("tiny"):
        cfg, B, N = WL.CONFIGS["tiny"], 32, int(case[-1])
        keys, offs = WL.gen_batch(cfg, 4, 0, 0, batch=B)
    elif case.startswith("corr"):
        cfg, B, N = WL.CONFIGS["tiny"].with_(table_rows=(3000,) * 4), 512, int(case[-1])
        keys, offs = WL.gen_correlated_batch(cfg, 2, 0, 0, groups=16, rho=0.7, batch=B)
    else:
        cfg = WL.CONFIGS["dlrm"].with_(table_rows=tuple(r // 50 for r in WL.CONFIGS["dlrm"].table_rows))
        B, N = 2048, 4
        keys, offs = WL.gen_batch(cfg, 1, 0, 0, batch=B)
    ctx = make_ctx(cfg, B, N=max(N, 2), K=len(keys))
    perm, mbo = ctx.fwp_schedule(to_dev(keys, torch.int64), to_dev(offs, torch.int32), B, N, "clustered")
    ref_perm, ref_mbo = OC.cluster_rounds(OC.sample_keysets(keys, offs, cfg.num_features), N)
    assert np.array_equal(perm.cpu().numpy(), ref_perm)
    assert np.array_equal(mbo.cpu().numpy(), ref_mbo)


def test_cluster_hand_worked_example_gpu():
    """R14 on the hand-worked multi-round example of
    tests/test_oracle_pins.py::test_cluster_rounds_hand_worked (admission sizes
    1, 1, 1, 2; ties broken by growth and by id): the GPU greedy gives the
    hand-derived partition."""
    from test_oracle_pins import HAND_KEYSETS, HAND_PERM
    cfg = WL.CONFIGS["tiny"].with_(table_rows=(64,), bag_len=(1, 4))
    keys = np.array([k for ks in HAND_KEYSETS for k in sorted(ks)], np.int64)     # table 0, row = key
    offs = np.concatenate([[0], np.cumsum([len(ks) for ks in HAND_KEYSETS])]).astype(np.int32)
    ctx = make_ctx(cfg, 12, N=2, K=len(keys))
    perm, mbo = ctx.fwp_schedule(to_dev(keys, torch.int64), to_dev(offs, torch.int32), 12, 2, "clustered")
    assert perm.cpu().numpy().tolist() == HAND_PERM
    assert mbo.cpu().numpy().tolist() == [0, 6, 12]


def test_cluster_repeated_batches_same_shape():
    """The captured round sequence is replayed for later batches of the same
    shape, including batches whose largest sample (smax, hence the number of
    rank-key bins) differs: every batch still matches the oracle."""
    cfg = WL.CONFIGS["tiny"].with_(table_rows=(3000,) * 4)
    long = cfg.with_(bag_len=(5, 8), bag_repeats=True)
    B, N = 512, 4
    ctx = make_ctx(cfg, B, N=N, K=B * cfg.num_features * long.bag_len[1])
    side = torch.cuda.Stream()   # a non-legacy stream: the rounds are captured and replayed
    for t in range(4):
        gen_cfg = cfg if t % 2 == 0 else long
        keys, offs = WL.gen_correlated_batch(gen_cfg, 9, t, 0, groups=8, rho=0.6, batch=B)
        kd, od = to_dev(keys, torch.int64), to_dev(offs, torch.int32)
        side.wait_stream(torch.cuda.current_stream())
        perm, mbo = ctx.fwp_schedule(kd, od, B, N, "clustered", stream=side)
        torch.cuda.synchronize()
        ref_perm, _ = OC.cluster_rounds(OC.sample_keysets(keys, offs, cfg.num_features), N)
        assert np.array_equal(perm.cpu().numpy(), ref_perm), t


def test_train_w1_clustered_p1_bit_exact():
    """Prop. 2 on the GPU: a clustered FWP window gives the Eq. 1 tables."""
    cfg = WL.CONFIGS["tiny"]
    B, N, T, F, d = 64, 4, 4, cfg.num_features, cfg.dim
    batches = [WL.gen_batch(cfg, 8, t, 0, batch=B) for t in range(T)]
    douts = [WL.gen_dout(8, t, 0, B * F, d, "dyadic") for t in range(T)]
    ctx = make_ctx(cfg, B, N=N, K=max(len(b[0]) for b in batches), init="dyadic", seed=11)
    run = Runner(ctx, N=N, schedule="clustered", pipelined=True, lr_over_B=2.0 ** -10)
    db = [(to_dev(k, torch.int64), to_dev(o, torch.int32), B) for k, o in batches]
    cap = B // N
    for t in range(T):
        def dout_fn(tt, i, pooled, t=t):
            perm = run.sched[t % 2][0].cpu().numpy()
            samples = perm[i * cap:(i + 1) * cap]
            bags = (samples[:, None] * F + np.arange(F)[None, :]).reshape(-1)
            return to_dev(douts[t][bags], torch.float32)
        outs = run.step(db[t], db[t + 1] if t + 1 < T else None, dout_fn)
        torch.cuda.synchronize()
        perm = run.sched[t % 2][0].cpu().numpy()
        tab_ref = OS.LazyTable(11, d, "dyadic")
        for tt in range(t + 1):
            res = OS.sync_step(tab_ref, [batches[tt]], [douts[tt]], 2.0 ** -10)
        pooled = np.concatenate([o.cpu().numpy() for o in outs])
        order = (perm[:, None] * F + np.arange(F)[None, :]).reshape(-1)
        assert np.array_equal(pooled, res.pooled[0][order])
    allk = np.unique(np.concatenate([b[0] for b in batches]))
    assert np.array_equal(ctx.read_rows(to_dev(allk, torch.int64)).cpu().numpy(), tab_ref.get(allk))


# --------------------------------------------------------------------------- edge cases
def _p1_check(cfg, batches, N, pipelined=True, lr=2.0 ** -10, seed=5, **ctx_kw):
    """Run the given per-step batches (W=1) and compare pooled rows of every
    step and the final rows bit-exactly against the oracle (P1)."""
    F, d = cfg.num_features, cfg.dim
    T = len(batches)
    douts = [WL.gen_dout(seed, t, 0, (len(o) - 1), d, "dyadic") for t, (k, o) in enumerate(batches)]
    B = (len(batches[0][1]) - 1) // F
    K = max(1, max(len(k) for k, _ in batches))
    ctx = make_ctx(cfg, B, N=N, K=K, init="dyadic", seed=seed, **ctx_kw)
    run = Runner(ctx, N=N, pipelined=pipelined, lr_over_B=lr)
    db = [(to_dev(k, torch.int64), to_dev(o, torch.int32), B) for k, o in batches]
    cap = B // N
    tab = OS.LazyTable(seed, d, "dyadic")
    for t in range(T):
        outs = run.step(db[t], db[t + 1] if t + 1 < T else None,
                        lambda tt, i, p, t=t: to_dev(douts[t][i * cap * F:(i + 1) * cap * F], torch.float32))
        torch.cuda.synchronize()
        res = OS.sync_step(tab, [batches[t]], [douts[t]], lr)
        assert np.array_equal(np.concatenate([o.cpu().numpy() for o in outs]), res.pooled[0]), t
    allk = np.unique(np.concatenate([k for k, _ in batches] + [np.zeros(1, np.int64)]))
    assert np.array_equal(ctx.read_rows(to_dev(allk, torch.int64)).cpu().numpy(), tab.get(allk))


def test_edge_empty_bags_empty_samples_and_single_sample_microbatches():
    """Empty bags pool to zero (reading Q5), an all-empty sample, micro-batches
    of one sample (N = B), and a step whose batch has no keys at all."""
    cfg = WL.CONFIGS["tiny"]
    F, B = cfg.num_features, 8
    batches = []
    for t in range(3):
        keys, offs = WL.gen_batch(cfg, 40 + t, t, 0, batch=B)
        lens = np.diff(offs).astype(np.int64)
        lens[::3] = 0                      # every third bag empty
        lens[F:2 * F] = 0                  # sample 1 has no keys
        new_off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
        new_keys = np.concatenate([keys[offs[b]:offs[b] + lens[b]] for b in range(B * F)])
        batches.append((new_keys.astype(np.int64), new_off))
    batches.append((np.zeros(0, np.int64), np.zeros(B * F + 1, np.int32)))   # no keys
    batches.append(batches[0])
    _p1_check(cfg, batches, N=8)
    _p1_check(cfg, batches, N=2, pipelined=False)


def test_edge_single_key_everywhere_hot():
    """Degenerate skew: every occurrence is the same key (one hot segment of
    B*F rows, split into chunks) plus the table-boundary rows."""
    cfg = WL.CONFIGS["tiny"].with_(bag_repeats=True)
    F, B = cfg.num_features, 64
    offs = np.arange(B * F + 1, dtype=np.int32) * 2
    keys = np.full(B * F * 2, (2 << 40) | 999, dtype=np.int64)
    keys[1::7] = (3 << 40) | 0
    _p1_check(cfg, [(keys, offs), (keys[::-1].copy(), offs)], N=4)


@pytest.mark.parametrize("d,N", [(16, 1), (128, 1), (128, 2)])
def test_edge_segments_cut_by_ranges_and_giant_segment(d, N):
    """The segment-sum works on fixed ranges of 256 sorted occurrences: one key
    with ~80K occurrences (hundreds of ranges: the block fix-up), keys of a few
    hundred occurrences (the lane-group fix-up), and many short keys cut by a
    range boundary.  N = 1 runs the fused update (frozen rows prefetched)."""
    cfg = WL.CONFIGS["tiny"].with_(dim=d, bag_repeats=True)
    F, B, L = cfg.num_features, 4096, 10
    rng = np.random.default_rng(7)
    offs = (np.arange(B * F + 1, dtype=np.int64) * L).astype(np.int32)
    K = B * F * L
    rows = rng.integers(0, 1000, size=K)
    tabs = rng.integers(0, 4, size=K)
    keys = (tabs.astype(np.int64) << 40) | rows
    keys[rng.random(K) < 0.5] = (1 << 40) | 17            # the giant segment
    keys[rng.random(K) < 0.02] = (2 << 40) | 3             # ~3K occurrences
    keys[rng.random(K) < 0.002] = (3 << 40) | 999          # ~330 occurrences
    keys2 = keys[::-1].copy()
    _p1_check(cfg, [(keys, offs), (keys2, offs)], N=N, lr=2.0 ** -12)


@pytest.mark.parametrize("d,N", [(16, 1), (128, 2)])
def test_edge_many_features_per_sample(d, N):
    """70 bags per sample (more than a lane group's 4..32 lanes hold at once:
    the streaming pool reloads its window of bag ends), empty bags included,
    bags of up to 5 keys on 3 tables (feature -> table map)."""
    cfg = WL.CONFIGS["tiny"].with_(table_rows=(3000, 700, 41), dim=d, bag_len=(0, 5), bag_repeats=True,
                                   feature_table=tuple(f % 3 for f in range(70)))
    batches = [WL.gen_batch(cfg, 80 + t, t, 0, batch=64) for t in range(3)]
    _p1_check(cfg, batches, N=N)


# --------------------------------------------------------------------------- soak
@pytest.mark.parametrize("N", [1, 2])
def test_long_run_soak_p1(N):
    """120 pipelined steps over 3 cycled batches of a small hot table (every
    key updated many times, slots and events reused 60 times each): pooled
    rows of every step and the final table bit-exact against the oracle (P1)."""
    cfg = WL.CONFIGS["tiny"].with_(table_rows=(400, 300, 200, 100), zipf=1.2, bag_repeats=True, dim=32)
    base = [WL.gen_batch(cfg, 90 + t, t, 0, batch=64) for t in range(3)]
    batches = [base[t % 3] for t in range(120)]
    _p1_check(cfg, batches, N=N, lr=2.0 ** -14)


# --------------------------------------------------------------------------- DBP stress
@pytest.mark.parametrize("p_reuse,zero_copy", [(0.7, "0"), (0.3, "0"), (0.7, "1")])
def test_dbp_stress_high_overlap_p1(monkeypatch, p_reuse, zero_copy):
    """BASELINE configs[3] structure at test size: one table feeding all 26
    features, batch t+1 reusing batch t's keys with probability p (the
    intersection I/U_o the refresh copies grows with p), 5 pipelined steps:
    pooled rows and final rows bit-exact (P1), the measured intersection
    matching the oracle's |K(t) cap K(t+1)|."""
    monkeypatch.setenv("NEST_ZERO_COPY", zero_copy)
    cfg = WL.CONFIGS["dbp_stress"].with_(table_rows=(200_000,), dim=32, batch_local=256)
    batches = WL.gen_overlap_batches(cfg, 11, 5, 0, p_reuse)
    inter = [len(np.intersect1d(batches[t][0], batches[t + 1][0])) / len(np.unique(batches[t + 1][0]))
             for t in range(4)]
    assert min(inter) > (0.6 if p_reuse > 0.5 else 0.3)
    _p1_check(cfg, batches, N=1, lr=2.0 ** -12)


# --------------------------------------------------------------------------- zero-copy retrieval
@pytest.mark.parametrize("N,d", [(1, 128), (1, 16), (2, 64)])
def test_zero_copy_retrieval_p1_bit_exact(monkeypatch, N, d):
    """NEST_ZERO_COPY=1 (W=1, N=1, HBM tables): no retrieval copy and no
    refresh -- the pool and the fused update read the shard in place -- and the
    pipelined steps still reach the synchronous result bit for bit (P1), hot
    segments and empty bags included; with N > 1 the buffered path runs."""
    monkeypatch.setenv("NEST_ZERO_COPY", "1")
    cfg = WL.CONFIGS["tiny"].with_(table_rows=(4000, 50, 9, 2000), zipf=1.3, bag_len=(0, 6), bag_repeats=True,
                                   dim=d)
    batches = [WL.gen_batch(cfg, 60 + t, t, 0, batch=128) for t in range(5)]
    _p1_check(cfg, batches, N=N)


def test_zero_copy_adagrad_matches_oracle(monkeypatch):
    """Zero-copy with the fused row-wise AdaGrad update (P2 tolerance)."""
    monkeypatch.setenv("NEST_ZERO_COPY", "1")
    cfg = WL.CONFIGS["tiny"].with_(table_rows=(3000, 700, 90, 20), zipf=1.2, bag_repeats=True, dim=32)
    B, F, d, T = 64, cfg.num_features, cfg.dim, 4
    batches = [WL.gen_batch(cfg, 70 + t, t, 0, batch=B) for t in range(T)]
    douts = [WL.gen_dout(70, t, 0, B * F, d, "realistic") for t in range(T)]
    gs, lr, eps = 1.0 / 64, 0.05, 1e-8
    ctx = make_ctx(cfg, B, K=max(len(k) for k, _ in batches), init="uniform", seed=4,
                   optimizer="rowwise_adagrad", adagrad_eps=eps)
    run = Runner(ctx, N=1, pipelined=True, adagrad=(gs, lr))
    db = [(to_dev(k, torch.int64), to_dev(o, torch.int32), B) for k, o in batches]
    for t in range(T):
        dd = to_dev(douts[t], torch.float32)
        run.step(db[t], db[t + 1] if t + 1 < T else None, lambda tt, i, p, dd=dd: dd)
    run.join()
    torch.cuda.synchronize()
    tab = OS.LazyTable(4, d, "uniform")
    opt = OS.RowwiseAdagrad(lr=lr, grad_scale=gs, eps=eps)
    for t in range(T):
        OS.sync_step(tab, [batches[t]], [douts[t]], 0.0, optimizer=opt)
    allk = np.unique(np.concatenate([k for k, _ in batches]))
    assert rel_rowwise_ok(ctx.read_rows(to_dev(allk, torch.int64)).cpu().numpy(), tab.get(allk))


# --------------------------------------------------------------------------- checked mode
@pytest.mark.parametrize("N", [1, 2])
def test_checked_mode_guard_bands(monkeypatch, N):
    """Checked mode (NEST_GUARD=1): after pipelined multi-step runs with hot
    segments, ragged bags and empty bags, every guard band after the workspace
    buffers is intact (no out-of-bounds write), and the check does detect a
    clobbered workspace (negative control)."""
    monkeypatch.setenv("NEST_GUARD", "1")
    cfg = WL.CONFIGS["tiny"].with_(table_rows=(4000, 50, 9, 2000), zipf=1.3, bag_len=(0, 6), bag_repeats=True,
                                   dim=64)
    batches = [WL.gen_batch(cfg, 40 + t, t, 0, batch=128) for t in range(4)]
    _p1_check(cfg, batches, N=N)
    ctx = make_ctx(cfg, 128, N=N, K=max(len(k) for k, _ in batches))
    run = Runner(ctx, N=N, pipelined=True, lr_over_B=2.0 ** -10)
    db = [(to_dev(k, torch.int64), to_dev(o, torch.int32), 128) for k, o in batches]
    F, d, cap = cfg.num_features, cfg.dim, 128 // N
    dd = torch.ones((128 * F, d), device=DEV)
    for t in range(4):
        run.step(db[t], db[t + 1] if t + 1 < 4 else None, lambda tt, i, p: dd[i * cap * F:(i + 1) * cap * F])
    run.join()
    torch.cuda.synchronize()
    assert ctx.check_guards() == 0
    ctx.work_mem.zero_()                      # negative control: clobber the workspace
    torch.cuda.synchronize()
    assert ctx.check_guards() > 0


# --------------------------------------------------------------------------- trained tower (NEXT-4)
def test_trained_tower_sgd_step_matches_definition():
    """NEXT-4 at W=1: one tower call with tower_train applies W0 - lr * G^T X0
    (L = 1: dW_0 = dY_0^T X_0 with dY_0 the fixed top gradient G) and returns
    dX_0 = G W0, both against fp64 products of the same bf16 operands."""
    cfg = WL.CONFIGS["tiny"]
    B, F, d, H, lr = 32, cfg.num_features, cfg.dim, 64, 0.01
    ctx = make_ctx(cfg, B, tower_layers=1, tower_hidden=H, tower_train=True, tower_lr=lr)
    g = torch.Generator(device=DEV).manual_seed(3)
    pooled = (torch.randn((B * F, d), generator=g, device=DEV) * 0.5).to(torch.bfloat16)
    dout = torch.empty((B * F, d), dtype=torch.float32, device=DEV)
    w0 = ctx.tower_read("weights", 0).cpu().double().numpy()
    G = ctx.tower_read("top_grad").cpu().double().numpy()[:B]
    ctx.tower_fwd_bwd(pooled, dout)
    ctx.join()
    torch.cuda.synchronize()
    # no update before nest_tower_step (the window's micro-batches accumulate)
    assert np.array_equal(ctx.tower_read("weights", 0).cpu().double().numpy(), w0)
    ctx.tower_step()
    ctx.join()
    torch.cuda.synchronize()
    w1 = ctx.tower_read("weights", 0).cpu().double().numpy()
    X = pooled.float().cpu().double().numpy().reshape(B, F * d)
    ref_w1 = w0 - lr * (G.T @ X)
    assert np.all(np.abs(w1 - ref_w1) <= 1e-5 * (np.abs(w0) + lr * (np.abs(G).T @ np.abs(X))) + 1e-7)
    ref_dx = G @ w0
    got_dx = dout.cpu().double().numpy().reshape(B, F * d)
    assert np.all(np.abs(got_dx - ref_dx) <= 1e-5 * (np.abs(G) @ np.abs(w0)) + 1e-7)
    assert not np.array_equal(w1, w0)
    # the fixed tower (default) leaves its weights alone
    ctx2 = make_ctx(cfg, B, tower_layers=1, tower_hidden=H)
    v0 = ctx2.tower_read("weights", 0).cpu().numpy()
    ctx2.tower_fwd_bwd(pooled, dout)
    ctx2.tower_step()
    ctx2.join()
    torch.cuda.synchronize()
    assert np.array_equal(ctx2.tower_read("weights", 0).cpu().numpy(), v0)


@pytest.mark.parametrize("L", [1, 3])
def test_trained_tower_micro_batches_accumulate(L):
    """ADVICE r01 / Prop. 2: with FWP the tower runs once per
    micro-batch, but the window's weights stay frozen and the batch makes ONE
    dense update -- N = 2 micro-batch calls + tower_step reach the weights of
    one full-batch call + tower_step (fp32 dW accumulation: same terms, other
    rounding order), and both micro-batches' input gradients use W0."""
    cfg = WL.CONFIGS["tiny"]
    B, F, d, H, lr = 32, cfg.num_features, cfg.dim, 64, 0.05
    g = torch.Generator(device=DEV).manual_seed(5)
    pooled = (torch.randn((B * F, d), generator=g, device=DEV) * 0.5).to(torch.bfloat16)
    res = []
    for N in (1, 2):
        ctx = make_ctx(cfg, B, tower_layers=L, tower_hidden=H, tower_train=True, tower_lr=lr)
        dout = torch.empty((B * F, d), dtype=torch.float32, device=DEV)
        rows = B * F // N
        for i in range(N):
            ctx.tower_fwd_bwd(pooled[i * rows:(i + 1) * rows], dout[i * rows:(i + 1) * rows])
        ctx.tower_step()
        ctx.join()
        torch.cuda.synchronize()
        res.append(([ctx.tower_read("weights", l).cpu().double().numpy() for l in range(L)],
                    dout.cpu().double().numpy()))
        w0 = make_ctx(cfg, B, tower_layers=L, tower_hidden=H, tower_train=True,
                      tower_lr=lr).tower_read("weights", 0).cpu().double().numpy()
        assert not np.allclose(res[-1][0][0], w0)
    (wa, da), (wb, db) = res
    for a, b in zip(wa, wb):
        assert np.allclose(a, b, rtol=1e-4, atol=1e-6), float(np.abs(a - b).max())
    # the input gradients of both micro-batches came from the same weights
    # (the top gradient is per row of the batch, so the halves match the full run)
    assert np.allclose(da, db, rtol=1e-3, atol=1e-5)


# --------------------------------------------------------------------------- host-DRAM tier
@pytest.mark.parametrize("N,pipelined,d", [(1, True, 16), (2, True, 16), (1, False, 128), (4, True, 128)])
def test_host_tier_p1_bit_exact(N, pipelined, d):
    """NEXT-3: the table shard in pinned host memory (retrieval, refresh and
    write-back over PCIe) reaches the same bits as the oracle -- and so as the
    HBM tier -- through the DBP/FWP pipeline, hot segments included."""
    cfg = WL.CONFIGS["tiny"].with_(table_rows=(4000, 50, 9, 2000), zipf=1.3, bag_repeats=True, dim=d)
    batches = [WL.gen_batch(cfg, 60 + t, t, 0, batch=512) for t in range(4)]
    _p1_check(cfg, batches, N=N, pipelined=pipelined, table_location="host")


def test_host_tier_rowwise_adagrad_matches_hbm():
    """Row-wise AdaGrad with the shard and its accumulators in host memory:
    bitwise the HBM-tier result (same kernels, same order)."""
    cfg = WL.CONFIGS["tiny"].with_(table_rows=(5000, 3000, 200, 77), zipf=1.3, bag_repeats=True, dim=32)
    B, T, F, d = 256, 4, cfg.num_features, cfg.dim
    batches = [WL.gen_batch(cfg, 9, t, 0, batch=B) for t in range(T)]
    douts = [to_dev(WL.gen_dout(9, t, 0, B * F, d, "realistic"), torch.float32) for t in range(T)]
    K = max(len(b[0]) for b in batches)
    res = []
    for loc in ("hbm", "host"):
        ctx = make_ctx(cfg, B, N=1, K=K, init="uniform", seed=4, optimizer="rowwise_adagrad", table_location=loc)
        run = Runner(ctx, N=1, pipelined=True, adagrad=(1.0 / B, 0.05))
        db = [(to_dev(k, torch.int64), to_dev(o, torch.int32), B) for k, o in batches]
        for t in range(T):
            run.step(db[t], db[t + 1] if t + 1 < T else None, lambda tt, i, p, dd=douts[t]: dd)
        run.join()
        torch.cuda.synchronize()
        allk = to_dev(np.unique(np.concatenate([b[0] for b in batches])), torch.int64)
        res.append((ctx.read_rows(allk).cpu().numpy(), ctx.read_state(allk).cpu().numpy()))
        ctx.close()
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])


def test_host_tier_pointer_kind_checked():
    """nest_create rejects device memory for the host tier and pinned host
    memory for the HBM tier (include/nest.h, table_location)."""
    import ctypes as C
    from paper_2604_06956_b200 import _lib as L
    lib = L.load()
    rows = (C.c_int64 * 4)(1000, 1000, 1000, 1000)
    work = None
    for loc, mem in ((L.TABLE_HOST, "cuda"), (L.TABLE_HBM, "pinned")):
        cfg = L.Config(world=1, rank=0, num_tables=4, dim=16, table_rows=rows, pooling=0, num_features=4,
                       max_keys=512, max_batch=32, max_micro_batches=1, seed=1, table_location=loc)
        tb, wb = C.c_size_t(), C.c_size_t()
        assert lib.nest_workspace_bytes(C.byref(cfg), C.byref(tb), C.byref(wb)) == 0
        tab = (torch.empty(tb.value, dtype=torch.uint8, device=DEV) if mem == "cuda"
               else torch.empty(tb.value, dtype=torch.uint8, pin_memory=True))
        work = torch.empty(wb.value, dtype=torch.uint8, device=DEV)
        ctx = C.c_void_p()
        st = lib.nest_create(C.byref(cfg), None, C.c_void_p(tab.data_ptr()), C.c_void_p(work.data_ptr()),
                             C.c_void_p(torch.cuda.current_stream(DEV).cuda_stream), C.byref(ctx))
        assert st == 1 and not ctx.value, (loc, mem, st)
        assert b"table_location" in lib.nest_last_error(None) or b"memory" in lib.nest_last_error(None)


# --------------------------------------------------------------------------- errors
def test_error_paths():
    cfg = WL.CONFIGS["tiny"]
    keys, offs = WL.gen_batch(cfg, 0, 0, 0, batch=32)
    ctx = make_ctx(cfg, 32, N=4)
    with pytest.raises(NestError) as e:
        ctx.fwp_schedule(None, None, 30, 4)
    assert e.value.status == "NEST_ERR_DIVISIBILITY"
    out = torch.empty((8 * 4, 16), device=DEV)
    with pytest.raises(NestError) as e:
        ctx.lookup_fwd(0, 0, out)
    assert e.value.status == "NEST_ERR_ORDER"
    bad = keys.copy()
    bad[5] = (2 << 40) | 5000          # row >= rows[2]
    with pytest.raises(NestError) as e:
        ctx.route(0, to_dev(bad, torch.int64), to_dev(offs, torch.int32), 32)
    assert e.value.status == "NEST_ERR_KEY_RANGE"
    with pytest.raises(NestError):     # sticky
        ctx.route(0, to_dev(keys, torch.int64), to_dev(offs, torch.int32), 32)


def test_route_split_and_window_misuse():
    """nest_route_begin / nest_route_end ordering, and the NCCL-free window
    rendezvous: out-of-order calls are NEST_ERR_ORDER, foreign or misordered
    records NEST_ERR_INVALID, checked-mode queries outside checked mode
    NEST_ERR_INVALID -- and a context stays usable after a host-side error."""
    cfg = WL.CONFIGS["tiny"]
    keys, offs = WL.gen_batch(cfg, 0, 0, 0, batch=32)
    kd, od = to_dev(keys, torch.int64), to_dev(offs, torch.int32)
    ctx = make_ctx(cfg, 32, N=2)
    with pytest.raises(NestError) as e:
        ctx.route_end(0)                               # no route begun
    assert e.value.status == "NEST_ERR_ORDER"
    ctx.route_begin(0, kd, od, 32)
    with pytest.raises(NestError) as e:
        ctx.route_begin(1, kd, od, 32)                 # scratch in use
    assert e.value.status == "NEST_ERR_ORDER"
    with pytest.raises(NestError) as e:
        ctx.fwp_schedule(kd, od, 32, 2, "clustered")   # scratch in use
    assert e.value.status == "NEST_ERR_ORDER"
    out = torch.empty((32 * cfg.num_features, cfg.dim), device=DEV)
    with pytest.raises(NestError) as e:
        ctx.lookup_fwd(0, 0, out)                      # slot not routed until route_end
    assert e.value.status == "NEST_ERR_ORDER"
    ctx.route_end(0)
    ctx.lookup_fwd(0, 0, out)                          # usable again
    torch.cuda.synchronize()
    ref = OS.forward(OS.LazyTable(1, cfg.dim, "dyadic"), keys, offs)
    assert np.array_equal(out.cpu().numpy(), ref)
    with pytest.raises(NestError) as e:
        ctx.check_guards()
    assert e.value.status == "NEST_ERR_INVALID"
    # NCCL-free world of 2 in one process: route before connect, bad records
    c0 = make_ctx(cfg, 32, world=2, rank=0)
    c1 = make_ctx(cfg, 32, world=2, rank=1)
    with pytest.raises(NestError) as e:
        c0.route(0, kd, od, 32)
    assert e.value.status == "NEST_ERR_ORDER"
    r0, r1 = c0.window_export(), c1.window_export()
    with pytest.raises(NestError) as e:
        c0.window_connect([r1, r0])                    # not in rank order
    assert e.value.status == "NEST_ERR_INVALID"
    c2 = make_ctx(cfg.with_(dim=32), 32, world=2, rank=1)
    with pytest.raises(NestError) as e:
        c0.window_connect([r0, c2.window_export()])    # another geometry
    assert e.value.status == "NEST_ERR_INVALID"
    c0.window_connect([r0, r1])
    with pytest.raises(NestError) as e:
        c0.window_connect([r0, r1])
    assert e.value.status == "NEST_ERR_ORDER"
    for c in (c2, c1, c0, ctx):
        c.close()


def test_refresh_required_after_pipelined_route():
    """Routing the next batch while the active slot's update is pending makes
    its gather skip K(t) (the refresh supplies those rows): a lookup of that
    slot before nest_dbp_refresh is an ordering error; after it, the rows are
    the updated ones (P1, bit-exact)."""
    cfg = WL.CONFIGS["tiny"]
    B, F, d = 32, cfg.num_features, cfg.dim
    b0, b1 = WL.gen_batch(cfg, 3, 0, 0, batch=B), WL.gen_batch(cfg, 3, 1, 0, batch=B)
    ctx = make_ctx(cfg, B, N=1, seed=6)
    k0, o0 = to_dev(b0[0], torch.int64), to_dev(b0[1], torch.int32)
    k1, o1 = to_dev(b1[0], torch.int64), to_dev(b1[1], torch.int32)
    out = torch.empty((B * F, d), device=DEV)
    ctx.route(0, k0, o0, B)
    ctx.lookup_fwd(0, 0, out)
    ctx.route(1, k1, o1, B)                     # window 0 still open: gather skips K(0)
    with pytest.raises(NestError) as e:
        ctx.lookup_fwd(1, 0, out)
    assert e.value.status == "NEST_ERR_ORDER"
    dout = to_dev(WL.gen_dout(3, 0, 0, B * F, d, "dyadic"), torch.float32)
    ctx.grad_bwd_update(0, 0, dout, 2.0 ** -10)
    ctx.dbp_refresh(0, 1)
    ctx.lookup_fwd(1, 0, out)
    torch.cuda.synchronize()
    tab = OS.LazyTable(6, d, "dyadic")
    OS.sync_step(tab, [b0], [dout.cpu().numpy()], 2.0 ** -10)
    ref = OS.sync_step(tab, [b1], [np.zeros((B * F, d))], 0.0).pooled[0]
    assert np.array_equal(out.cpu().numpy(), ref)


# --------------------------------------------------------------------------- full size
def test_genrec_full_tables_unpooled_sampled():
    """BASELINE configs[2] (8 x 50M rows, d=64, seq 1,024 unpooled, Zipf 1.2) with
    the full table sizes and a reduced batch: expanded rows and updated rows
    checked one by one against the oracle's PRF rows and per-key gradients."""
    cfg = WL.CONFIGS["genrec"]
    B, N, F, d = 128, 2, cfg.num_features, cfg.dim
    keys, offs = WL.gen_batch(cfg, 0, 0, 0, batch=B)
    U = len(np.unique(keys))
    ctx = NestContext(cfg.table_rows, d, pooling="none", max_keys=len(keys), max_batch=B,
                      max_micro_batches=N, max_recv_keys=U + 16, max_mb_rows=2 * U + 16,
                      seed=9, init_mode="uniform", device=DEV)
    run = Runner(ctx, N=N, pipelined=False, lr_over_B=0.25)
    kd, od = to_dev(keys, torch.int64), to_dev(offs, torch.int32)
    dout_all = torch.randn(len(keys), d, device=DEV, generator=torch.Generator(DEV).manual_seed(1))
    cap = B // N
    mb_occ = [(int(offs[i * cap * F]), int(offs[(i + 1) * cap * F])) for i in range(N)]
    outs = run.step((kd, od, B), None, lambda t, i, p: dout_all[mb_occ[i][0]:mb_occ[i][1]])
    torch.cuda.synchronize()
    v = ctx.route_view(0)
    assert v["info"].uniq == U and np.array_equal(v["uniq"][v["inverse"]], keys)
    rng = np.random.default_rng(2)
    for j in rng.integers(0, len(keys), size=64):      # expanded occurrence rows
        i = 0 if j < mb_occ[0][1] else 1
        got = outs[i][j - mb_occ[i][0]].cpu().numpy()
        assert np.array_equal(got, OPRF.init_rows(9, keys[j:j + 1], d)[0])
    dnp = dout_all.cpu().numpy().astype(np.float64)
    sample = rng.choice(np.unique(keys), size=48, replace=False)
    got = ctx.read_rows(to_dev(sample, torch.int64)).cpu().numpy()
    for k, row in zip(sample, got):
        occ = np.nonzero(keys == k)[0]
        ref = OS.sgd_rows(OPRF.init_rows(9, np.array([k]), d), dnp[occ].sum(axis=0)[None], 0.25)[0]
        scale = np.abs(dnp[occ]).sum(axis=0) * 0.25 + np.abs(ref)
        assert np.all(np.abs(row - ref) <= 1e-5 * scale + 1e-7)
    ctx.close()


def test_dlrm_full_size_bench_path_p1_every_row():
    """BASELINE configs[1] (26 tables, 103.3M rows, d=128, 65,536 samples) at
    W=1 on the bench's exact call path -- pipelined DBP (route of t+1 on the
    aux lane, prefetch gather skipping the pending update's keys + refresh),
    nest_lookup_fwd_bf16 (bf16 pooled rows for the dense consumer), the fused
    segment-sum + SGD of N=1 -- for 3 steps in regime P1 (dyadic rows and
    gradients, s = 2^-12: every sum exact in fp32).  EVERY pooled row of every
    step equals bf16(oracle pooled) bit for bit, and EVERY row touched by the 3
    steps equals the oracle's E_3 bit for bit (oracle.step.sync_step)."""
    cfg = WL.CONFIGS["dlrm"]
    B, F, d, T, lr = cfg.batch_local, cfg.num_features, cfg.dim, 3, 2.0 ** -12
    batches = [WL.gen_batch(cfg, 7, t, 0) for t in range(T)]
    douts = [WL.gen_dout(7, t, 0, B * F, d, "dyadic") for t in range(T)]
    K = max(len(k) for k, _ in batches)
    ctx = NestContext(cfg.table_rows, d, max_keys=K, max_batch=B, seed=9, init_mode="dyadic", device=DEV)
    run = Runner(ctx, N=1, pipelined=True, lr_over_B=lr, pooled_dtype=torch.bfloat16)
    db = [(to_dev(k, torch.int64), to_dev(o, torch.int32), B) for k, o in batches]
    got_pooled = []
    for t in range(T):
        dd = to_dev(douts[t], torch.float32)
        outs = run.step(db[t], db[t + 1] if t + 1 < T else None, lambda tt, i, p, dd=dd: dd)
        run.join()
        torch.cuda.synchronize()
        assert outs[0].dtype == torch.bfloat16
        got_pooled.append(outs[0].cpu().view(torch.int16).numpy())
        del dd
    touched = np.unique(np.concatenate([k for k, _ in batches]))
    got_rows = ctx.read_rows(to_dev(touched, torch.int64)).cpu().numpy()
    ctx.close()
    tab = OS.LazyTable(9, d, "dyadic")
    for t in range(T):
        res = OS.sync_step(tab, [batches[t]], [douts[t]], lr)
        ref = torch.from_numpy(res.pooled[0]).to(torch.bfloat16).view(torch.int16).numpy()
        bad = np.nonzero((got_pooled[t] != ref).any(axis=1))[0]
        assert len(bad) == 0, f"step {t}: {len(bad)} pooled rows differ, first {bad[:5]}"
    ref_rows = tab.get(touched)
    bad = np.nonzero((got_rows != ref_rows).any(axis=1))[0]
    assert len(bad) == 0, f"{len(bad)} of {len(touched)} touched rows differ"


@pytest.mark.parametrize("N", [1, 4])
def test_dlrm_full_size_w1_sampled(N):
    """BASELINE configs[1] at W=1 (N = 1 is the bench launch configuration:
    fused segment-sum + update): routing invariants at full size, sampled
    pooled rows and sampled updated rows -- the hottest keys included --
    computed one by one by the oracle."""
    cfg = WL.CONFIGS["dlrm"]
    B, F, d = cfg.batch_local, cfg.num_features, cfg.dim
    keys, offs = WL.gen_batch(cfg, 0, 0, 0)
    ctx = NestContext(cfg.table_rows, d, max_keys=len(keys), max_batch=B, max_micro_batches=N,
                      seed=5, init_mode="uniform", device=DEV)
    run = Runner(ctx, N=N, pipelined=False, lr_over_B=0.5)
    kd, od = to_dev(keys, torch.int64), to_dev(offs, torch.int32)
    cap = B // N
    dout_all = torch.randn(B * F, d, device=DEV, generator=torch.Generator(DEV).manual_seed(0))
    outs = run.step((kd, od, B), None, lambda t, i, p: dout_all[i * cap * F:(i + 1) * cap * F])
    torch.cuda.synchronize()
    v = ctx.route_view(0)
    info = v["info"]
    # routing invariants at full size
    assert info.uniq == len(np.unique(keys))
    assert (np.diff(v["uniq"]) > 0).all()
    assert np.array_equal(v["uniq"][v["inverse"]], keys)
    # sampled pooled rows: oracle computes each bag from PRF rows
    rng = np.random.default_rng(0)
    for q in rng.integers(0, B * F, size=64):
        i, r = divmod(int(q), cap * F)
        b, f = i * cap + r // F, r % F
        bag = keys[offs[b * F + f]:offs[b * F + f + 1]]
        ref = OS.pool_sum(OPRF.init_rows(5, bag, d), np.array([0, len(bag)]))[0]
        assert rel_rowwise_ok(outs[i][r][None].cpu().numpy(), ref[None])
    # sampled updated rows: e' = e0 - s * sum of the bag grads of its occurrences
    dnp = dout_all.cpu().numpy().astype(np.float64)
    bag_of = np.repeat(np.arange(B * F), np.diff(offs))
    uk, cnt = np.unique(keys, return_counts=True)
    sample = np.concatenate([uk[np.argsort(-cnt)[:8]], rng.choice(uk, size=64, replace=False)])
    got = ctx.read_rows(to_dev(sample, torch.int64)).cpu().numpy()
    order = np.argsort(keys, kind="stable")
    starts = np.searchsorted(keys[order], sample)
    for k, row, s0 in zip(sample, got, starts):
        occ = order[s0:s0 + cnt[np.searchsorted(uk, k)]]
        assert (keys[occ] == k).all()
        g = dnp[bag_of[occ]].sum(axis=0)
        ref = OS.sgd_rows(OPRF.init_rows(5, np.array([k]), d), g[None], 0.5)[0]
        scale = np.abs(dnp[bag_of[occ]]).sum(axis=0) * 0.5 + np.abs(ref)
        assert np.all(np.abs(row - ref) <= 1e-5 * scale + 1e-7)
