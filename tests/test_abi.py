"""The C-ABI library loads without a GPU, exports every symbol include/parm_b200.h declares with the
ABI version the binding expects, and rejects bad arguments before touching the device — CPU only."""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

import pytest

from paper_2407_00599_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "parm_b200.h"


def header_functions() -> list[str]:
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_]+\*?\s+\*?(parm_[a-z0-9_]+)\(", text, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2407_00599_b200 import build

    build.build()
    return _lib.load()


def test_header_lists_the_boundary():
    fns = header_functions()
    for required in ("parm_gate_fwd", "parm_gate_counts_bytes", "parm_route_dispatch", "parm_combine_fwd",
                     "parm_dispatch_bwd", "parm_esp_sum", "parm_gate_wgrad",
                     "parm_gemm", "parm_last_error", "parm_abi_version",
                     "parm_combine_fwd_fan", "parm_dispatch_bwd_fan", "parm_peer_barrier", "parm_push_rows",
                     "parm_fan_copy", "parm_gemm_peer", "parm_combine_bwd_dispatch"):
        assert required in fns


def test_every_declared_symbol_is_exported_and_typed(lib):
    fns = header_functions()
    assert set(fns) == set(_lib.SIGNATURES), "ctypes binding and header disagree"
    for name in fns:
        assert hasattr(lib, name), f"{name} missing from libparm_b200.so"
    assert lib.parm_abi_version() == _lib.ABI_VERSION
    m = re.search(r"#define PARM_ABI_VERSION (\d+)", HEADER.read_text())
    assert int(m.group(1)) == _lib.ABI_VERSION


def test_struct_layouts_match_header(lib):
    assert ctypes.sizeof(_lib.SlotViewC) == 8 + 4 * 4 + 5 * 8 + 8 * 8 + 2 * 4
    assert ctypes.sizeof(_lib.RowFanC) == 8 * 8 + 8
    assert ctypes.sizeof(_lib.IntFanC) == 8 * 8
    assert ctypes.sizeof(_lib.PeerSignalC) == 8 * 8 + 8 + 8 + 8
    assert ctypes.sizeof(_lib.RowsC) == 8 + 4 * 8
    assert ctypes.sizeof(_lib.GemmDescC) == 12 * 4 + 4 * ctypes.sizeof(_lib.RowsC) + 8


def _expect_arg_error(fn, *args, match):
    rc = fn(*args)
    assert rc == 1
    assert re.search(match, _lib.load().parm_last_error().decode())


def test_argument_validation_without_a_gpu(lib):
    # validation happens on the host before any launch, with the reference's error wording
    _expect_arg_error(lib.parm_gate_fwd, None, 8, None, 4, 8, 2, 3, None, None, None, None, None,
                      match=r"top_k \(3\) exceeds number of experts \(2\)")
    _expect_arg_error(lib.parm_route_dispatch, None, 8, None, None, 16, 9, 8, 4, 8, None, None, None, 0, 4, None, 8,
                      8, None, None, None, match="route_dispatch: need 1 <= k")
    _expect_arg_error(lib.parm_route_dispatch, None, 10, None, None, 16, 2, 8, 4, 10, None, None, None, 0, 4, None,
                      10, 10, None, None, None, match="counts/slot_idx/slot_src/fill required")
    _expect_arg_error(lib.parm_route_dispatch, 16, 10, None, 32, 16, 2, 8, 4, 10, 64, 64, 64, 0, 4, None, 10, 10,
                      None, None, None, match="16-byte aligned")
    _expect_arg_error(lib.parm_combine_fwd, None, None, None, None, 4, 1, 8, None, 8, None,
                      match="null slot view")
    _expect_arg_error(lib.parm_combine_bwd_dispatch, None, 8, None, None, None, None, None, 4, 2, 4, 8, None, 0, 4,
                      None, None, 8, 8, None, None, match="null slot view")
    y = _lib.SlotViewC()
    y.ptr, y.e_local, y.n_p, y.slot_div = 4096, 4, 1, 1 << 30
    _expect_arg_error(lib.parm_combine_bwd_dispatch, None, 8, ctypes.byref(y), None, None, None, None, 4, 2, 4, 8,
                      None, 0, 4, None, None, 8, 8, None, None, match="combine weights and fill required")
    desc = _lib.GemmDescC()
    desc.kind = 7
    _expect_arg_error(lib.parm_gemm, ctypes.byref(desc), None, match="bad kind")
    desc.kind, desc.groups, desc.nhi, desc.nlo, desc.seg_len, desc.N, desc.K = 0, 1, 1, 1, 16, 100, 64
    _expect_arg_error(lib.parm_gemm, ctypes.byref(desc), None, match="N=100")


def test_gate_wgrad_workspace_query(lib):
    assert lib.parm_gate_wgrad_workspace(8192, 1024, 8) == 148 * 1024 * 8 * 4 + 16   # one partial per SM + barrier
    assert lib.parm_gate_counts_bytes(8192, 8) == 1024 * 8 * 4                    # 8-token tiles


def test_missing_library_fails_loudly(tmp_path):
    with pytest.raises(ImportError, match="no CPU fallback"):
        _lib.load(tmp_path / "nope.so")
