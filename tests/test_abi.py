"""The C-ABI library loads and exports every symbol include/nest.h declares
(no compute calls: runs without a GPU)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2604_06956_b200 import build as B
    B.build()
    from paper_2604_06956_b200 import _lib as L
    return L.load()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "nest.h")).read()
    return sorted(set(re.findall(r"NEST_API\s+[\w\s\*]+?\b(nest_\w+)\s*\(", src)))


def test_header_declares_expected_api():
    from paper_2604_06956_b200 import _lib as L
    assert declared_symbols() == sorted(L.SYMBOLS)


def test_every_declared_symbol_exported(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_host_only_calls(lib):
    from paper_2604_06956_b200 import _lib as L
    rows = (C.c_int64 * 4)(1000, 1000, 1000, 1001)
    cfg = L.Config(world=2, rank=1, num_tables=4, dim=16, table_rows=rows, pooling=0,
                   num_features=4, max_keys=1000, max_batch=64, max_micro_batches=4, seed=1)
    tb, wb = C.c_size_t(), C.c_size_t()
    assert lib.nest_workspace_bytes(C.byref(cfg), C.byref(tb), C.byref(wb)) == 0
    # rank 1 of 2 owns the odd rows: 500 + 500 + 500 + 500
    assert lib.nest_shard_rows(C.byref(cfg)) == 2000
    assert tb.value == 2000 * 16 * 4 and wb.value > 0
    cfg.dim = 48
    assert lib.nest_workspace_bytes(C.byref(cfg), C.byref(tb), C.byref(wb)) == 1  # INVALID
    assert b"dim" in lib.nest_last_error(None)
    cfg.dim = 16
    cfg.table_location = L.TABLE_HOST      # host-DRAM tier: same sizes
    assert lib.nest_workspace_bytes(C.byref(cfg), C.byref(tb), C.byref(wb)) == 0
    assert tb.value == 2000 * 16 * 4
    cfg.table_location = 7
    assert lib.nest_workspace_bytes(C.byref(cfg), C.byref(tb), C.byref(wb)) == 1  # INVALID
    assert b"table_location" in lib.nest_last_error(None)
    # tower width checked before any collective initialisation (nest_create)
    cfg.table_location = L.TABLE_HBM
    cfg.tower_layers, cfg.tower_hidden = 2, 8
    assert lib.nest_workspace_bytes(C.byref(cfg), C.byref(tb), C.byref(wb)) == 1  # INVALID
    assert b"tower_hidden" in lib.nest_last_error(None)
    cfg.tower_layers = 0
    assert lib.nest_version().startswith(b"nestpipe")


def test_sm100a_cubin_present():
    """The library carries sm_100a SASS (no PTX-only JIT path)."""
    import subprocess
    from paper_2604_06956_b200 import build as B
    B.build()
    out = subprocess.run(["cuobjdump", "--list-elf", B.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


# every struct of include/nest.h and its ctypes mirror in _lib.py
_STRUCTS = {"nest_config_t": "Config", "nest_slot_info_t": "SlotInfo", "nest_route_view_t": "RouteView",
            "nest_window_rec_t": "WindowRec", "nest_exchange_plan_t": "ExchangePlan",
            "nest_profile_stage_t": "ProfileStage", "nest_profile_summary_t": "ProfileSummary",
            "nest_profile_record_t": "ProfileRecord"}


def test_ctypes_mirrors_match_the_header(tmp_path):
    """sizeof and every field offset of the header's structs, compiled by gcc,
    equal the ctypes mirrors the binding passes through the ABI."""
    import shutil
    import subprocess
    from paper_2604_06956_b200 import _lib as L
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "nest.h"', "int main(void) {"]
    for cname, pyname in _STRUCTS.items():
        lines.append(f'printf("{cname} sizeof %zu\\n", sizeof({cname}));')
        for f in getattr(L, pyname)._fields_:
            lines.append(f'printf("{cname} {f[0]} %zu\\n", offsetof({cname}, {f[0]}));')
    lines += ["return 0;", "}"]
    src = tmp_path / "abi.c"
    src.write_text("\n".join(lines) + "\n")
    exe = tmp_path / "abi"
    subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = {}
    for ln in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.splitlines():
        s, f, v = ln.split()
        got[(s, f)] = int(v)
    for cname, pyname in _STRUCTS.items():
        py = getattr(L, pyname)
        assert got[(cname, "sizeof")] == C.sizeof(py), cname
        for f in py._fields_:
            assert got[(cname, f[0])] == getattr(py, f[0]).offset, (cname, f[0])
