"""Host-side bench.py arithmetic (no GPU): the roofline and whole-step HBM
fractions are algorithmic bytes over event time against the peak, the CPU
model string is read, and the tiny oracle baseline runs 10 steps."""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _stages(**kw):
    names = ["schedule", "route", "sort", "key_a2a", "owner_dedup", "gather", "refresh", "send_gather",
             "emb_a2a", "pool", "tower", "segsum", "grad_a2a", "update", "tower_dw", "emb_repush"]
    st = {n: {"records": 0, "ms": 0.0, "bytes": 0.0, "units": 0.0, "launches": 0, "hbm_bytes": 0.0} for n in names}
    for n, v in kw.items():
        ms, by = v[:2]
        st[n] = {"records": 10, "ms": ms, "bytes": by, "units": 0.0, "launches": 10,
                 "hbm_bytes": v[2] if len(v) > 2 else by}
    return st


def test_roofline_picks_the_longest_hbm_stage(monkeypatch):
    monkeypatch.setattr(bench, "peaks", lambda: (6000.0, 1400.0, "measured"))
    st = _stages(pool=(3.0, 12e9), segsum=(6.0, 24e9), tower=(20.0, 1e12))   # the tower is not an HBM stage
    r = bench.roofline_from(st, "x/W1/N1")
    assert r["kernel"] == "segsum"
    assert r["achieved"] == pytest.approx(24e9 / (6.0 * 1e6))            # bytes / (ms * 1e6) = GB/s
    assert r["frac"] == pytest.approx(r["achieved"] / 6000.0)
    assert r["bytes_per_launch"] == pytest.approx(24e9 / 10)
    assert r["ms_per_launch"] == pytest.approx(0.6)


def test_whole_step_hbm_sums_every_hbm_stage(monkeypatch):
    monkeypatch.setattr(bench, "peaks", lambda: (5000.0, 1400.0, "measured"))
    st = _stages(route=(1.0, 1e9), sort=(1.0, 2e9), gather=(1.0, 3e9), pool=(1.0, 4e9), segsum=(1.0, 5e9),
                 emb_a2a=(1.0, 9e9, 0.0))                                   # NVLink bytes are not counted
    w = bench.whole_step_hbm(st, steps=10, ms_step=2.0)
    assert w["bytes_per_step"] == pytest.approx(15e9 / 10)
    assert w["gbs"] == pytest.approx(1.5e9 / 2e6)
    assert w["frac"] == pytest.approx(w["gbs"] / 5000.0)
    assert "emb_a2a" not in w["stages"]


def test_whole_step_hbm_counts_the_local_side_of_fused_transports(monkeypatch):
    # W > 1: the fused segment-sum -> peer-store stage (grad_a2a) and the send
    # push (emb_a2a) move NVLink bytes (`bytes`) and local HBM bytes
    # (`hbm_bytes`); only the latter count towards the HBM fraction
    monkeypatch.setattr(bench, "peaks", lambda: (5000.0, 1400.0, "measured"))
    st = _stages(pool=(1.0, 4e9), update=(1.0, 2e9), grad_a2a=(1.0, 7e9, 3e9), emb_a2a=(1.0, 9e9, 1e9),
                 key_a2a=(1.0, 5e8, 0.0))
    w = bench.whole_step_hbm(st, steps=10, ms_step=2.0)
    assert w["bytes_per_step"] == pytest.approx((4e9 + 2e9 + 3e9 + 1e9) / 10)
    assert set(w["stages"]) == {"pool", "update", "grad_a2a", "emb_a2a"}


def test_cpu_model_and_tiny_oracle_baseline():
    assert isinstance(bench.cpu_model(), str) and bench.cpu_model()
    t = bench.tiny_oracle_baseline(0, steps=2)
    assert t["steps"] == 2 and t["value"] > 0 and "tiny" in t["sample"]
    json.dumps(t)


def test_clock_samples_are_taken_inside_the_timed_region(tmp_path):
    """bench.Clocks keeps the nvidia-smi samples whose timestamps fall inside
    the marked timed region (the nearest one if none does) and reports the
    throttle reasons seen there."""
    import datetime

    def line(t, sm, reasons=("Not Active",) * 4):
        ts = datetime.datetime.fromtimestamp(t).strftime("%Y/%m/%d %H:%M:%S.%f")[:-3]
        return ", ".join([ts, "0", str(sm), "1965", "900.0", "0x0"] + list(reasons)) + "\n"

    c = bench.Clocks(0)
    c.path = str(tmp_path / "clk.csv")
    t = 1_700_000_000.0
    with open(c.path, "w") as f:
        f.write(line(t - 1.0, 1200, ("Active", "Not Active", "Not Active", "Not Active")))   # warm-up
        f.write(line(t + 0.10, 1900))
        f.write(line(t + 0.15, 1950, ("Not Active", "Not Active", "Not Active", "Active")))
        f.write(line(t + 5.0, 1000))                                                           # after

    class _P:
        def terminate(self):
            pass

        def wait(self, timeout=None):
            return 0

    c.proc, c.f = _P(), open(str(tmp_path / "sink"), "w")
    c.t0, c.t1 = t, t + 0.2
    r = c.stop()
    assert r["samples"] == 2 and r["samples_in_timed_region"] == 2
    assert r["sm_mhz"] == pytest.approx(1925.0) and r["reasons"] == ["sw_power_cap"]
    # a region between two samples: the nearest sample stands in
    c.proc, c.f = _P(), open(str(tmp_path / "sink2"), "w")
    c.t0, c.t1 = t + 0.16, t + 0.17
    r = c.stop()
    assert r["samples"] == 1 and r["samples_in_timed_region"] == 0 and r["sm_mhz"] == 1950.0


def test_config_json_names_the_workload_and_exchanges(monkeypatch):
    import argparse
    import workload as WL
    monkeypatch.delenv("NEST_A2A", raising=False)
    monkeypatch.setenv("NEST_DIRECT_WB", "0")
    args = argparse.Namespace(micro_batches=1, schedule="sequential", optimizer="sgd", variant="et")
    cfg = WL.CONFIGS["dlrm"]
    one = bench.config_json(args, cfg, 1)
    two = bench.config_json(args, cfg, 2)
    assert one["workload"] == "dlrm" and one["exchanges"] is None and one["global_batch"] == cfg.batch_local
    assert two["global_batch"] == 2 * cfg.batch_local
    assert "fused" in two["exchanges"] and "direct write-back: off" in two["exchanges"]
    json.dumps(two)
