"""The C-ABI library loads on a machine without a GPU and exports exactly what
include/fsa_b200.h declares (no compute calls here)."""

import ctypes as C
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "fsa_b200.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fsa_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2511_13645_b200 import _build, _lib
    _build.build()
    return _lib.load()


def test_header_declares_the_operator_surface():
    names = declared_functions()
    for must in ("fsa_fused_1hop_fwd", "fsa_fused_2hop_fwd", "fsa_fused_1hop_bwd", "fsa_fused_2hop_bwd",
                 "fsa_ws_bytes", "fsa_derive_states", "fsa_xorshift_steps"):
        assert must in names


def test_every_declared_symbol_is_exported(lib):
    from paper_2511_13645_b200 import _lib
    names = declared_functions()
    assert sorted(_lib.SIGNATURES) == names, "ctypes table and header disagree"
    for n in names:
        assert hasattr(lib, n), n


def test_host_only_entry_points(lib):
    from paper_2511_13645_b200 import _lib
    assert b"sm_100a" in lib.fsa_version()
    assert lib.fsa_status_string(0) == b"ok"
    assert lib.fsa_status_string(_lib.FSA_ERR_WORKSPACE) == b"workspace too small"
    F32, F64 = _lib.FSA_F32, _lib.FSA_F64
    for op, args in ((_lib.FSA_OP_FWD1, (1024, 10, 0, 0, 0, 0)), (_lib.FSA_OP_FWD2, (1024, 15, 10, 0, 0, 0)),
                     (_lib.FSA_OP_BWD1, (1024, 10, 0, 100, F32, 10000)),
                     (_lib.FSA_OP_BWD2, (1024, 15, 10, 100, F32, 2449029))):
        assert lib.fsa_ws_bytes(op, *args) > 0
    assert lib.fsa_ws_bytes(_lib.FSA_OP_FWD2, 1024, 15, 0, 0, 0, 0) == 0  # k2 < 1
    assert lib.fsa_ws_bytes(_lib.FSA_OP_BWD2, 64, 4, 4, 0, F32, 100) == 0  # D < 1
    assert lib.fsa_ws_bytes(_lib.FSA_OP_BWD2, 64, 4, 4, 8, 99, 100) == 0  # bad dtype
    # bwd workspace grows with N (persistent per-node counters) and with the term table (G x D)
    assert lib.fsa_ws_bytes(_lib.FSA_OP_BWD2, 64, 4, 4, 8, F32, 10**6) > lib.fsa_ws_bytes(_lib.FSA_OP_BWD2, 64, 4, 4, 8, F32, 10)
    small = lib.fsa_ws_bytes(_lib.FSA_OP_BWD2, 64, 4, 4, 8, F32, 10)
    assert lib.fsa_ws_bytes(_lib.FSA_OP_BWD2, 64, 4, 4, 8 + 256, F32, 10) >= small + 64 * 4 * 256 * 4
    assert lib.fsa_ws_bytes(_lib.FSA_OP_BWD2, 64, 4, 4, 256, F64, 10) > lib.fsa_ws_bytes(_lib.FSA_OP_BWD2, 64, 4, 4, 256, F32, 10)


def test_argument_errors_are_reported_before_any_cuda_call(lib):
    from paper_2511_13645_b200 import _lib
    # null graph pointers / bad fanout / bad dtype are rejected on the host
    st = lib.fsa_fused_2hop_fwd(None, None, 10, None, 0, 0, 0, None, 4, 0, 2, 2, 1, 1,
                                None, None, None, None, None, 0, None, 0, None)
    assert st == _lib.FSA_ERR_ARG
    st = lib.fsa_fused_1hop_fwd(1, 1, 10, 1, 4, 4, 99, 1, 4, 0, 2, 1, 0, None, None, 1, 4, 1, 1 << 20, None)
    assert st == _lib.FSA_ERR_DTYPE
    st = lib.fsa_fused_1hop_fwd(1, 1, 10, 1, 4, 4, 0, 1, 4, 0, 0, 1, 0, None, None, 1, 4, 1, 1 << 20, None)
    assert st == _lib.FSA_ERR_ARG


def test_product_package_does_not_import_the_oracle():
    pkg = ROOT / "paper_2511_13645_b200"
    for py in pkg.rglob("*.py"):
        src = py.read_text()
        assert "from oracle" not in src and "import oracle" not in src, py


def test_tune_knobs_validate_arguments(lib):
    """fsa_tune: unknown knobs and out-of-range values are argument errors; the host-side knobs
    (3: re-zero CTAs, 4: count CTAs, 5: multi-hit CTAs, 6: first-hop path) set without a device
    and restore."""
    from paper_2511_13645_b200 import _lib
    assert lib.fsa_tune(99, 1) == _lib.FSA_ERR_ARG
    assert lib.fsa_tune(1, -1) == _lib.FSA_ERR_ARG
    assert lib.fsa_tune(2, 7) == _lib.FSA_ERR_ARG
    for knob, bad, default in ((3, 9, 1), (4, 65, 8), (5, 9, 0), (5, -1, 0), (6, 3, 1), (6, 0, 1)):
        assert lib.fsa_tune(knob, bad) == _lib.FSA_ERR_ARG
        assert lib.fsa_tune(knob, default) == _lib.FSA_OK


def test_first_hop_path_choice_by_mean_degree(monkeypatch):
    """The Python layer picks the 2-hop forward's first-hop path per graph: warp per root below
    HOP1_TILE_MEAN_DEGREE arcs per node, the tile sampler above; FSA_HOP1 pins it."""
    import torch
    from paper_2511_13645_b200 import fused
    from paper_2511_13645_b200.graph import CsrGraph

    calls = []

    class Lib:
        def fsa_tune(self, what, value):
            calls.append((what, value))
            return 0

    monkeypatch.setattr(fused._lib, "load", lambda *a, **k: Lib())
    monkeypatch.delenv("FSA_HOP1", raising=False)
    fused._hop1_set[0] = None

    def graph(n, e):
        rp = torch.zeros(n + 1, dtype=torch.int32)
        rp[1:] = e // n
        return CsrGraph(n, rp, torch.zeros(e, dtype=torch.int32))

    fused._select_hop1(graph(100, 5_000))      # mean 50: warp per root
    fused._select_hop1(graph(100, 5_000))      # unchanged: no second call
    fused._select_hop1(graph(100, 50_000))     # mean 500: tiles
    assert calls == [(6, 1), (6, 2)]
    monkeypatch.setenv("FSA_HOP1", "1")
    fused._select_hop1(graph(100, 5_000))      # pinned: left alone
    assert calls == [(6, 1), (6, 2)]
    fused._hop1_set[0] = None
