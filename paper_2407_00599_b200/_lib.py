"""ctypes binding of the C ABI in ``include/parm_b200.h`` (``libparm_b200.so``).

This is the only way the host layer reaches the GPU kernels.  There is no
fallback: if the library is missing or cannot load, every op raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libparm_b200.so"

_c_int = ctypes.c_int
_c_ll = ctypes.c_longlong
_vp = ctypes.c_void_p
_size = ctypes.c_size_t


MAX_PEERS = 8


class SlotViewC(ctypes.Structure):
    _fields_ = [
        ("ptr", _vp),
        ("e_local", _c_int),
        ("n_p", _c_int),
        ("slot_div", _c_int),
        ("n_peer", _c_int),
        ("stride_ep", _c_ll),
        ("stride_i", _c_ll),
        ("stride_p", _c_ll),
        ("stride_shi", _c_ll),
        ("stride_slo", _c_ll),
        ("peer", _vp * MAX_PEERS),
        ("peer_ep", _c_int),
        ("peer_p", _c_int),
    ]


class RowFanC(ctypes.Structure):
    _fields_ = [("ptr", _vp * MAX_PEERS), ("n", _c_int), ("pad_", _c_int)]


class IntFanC(ctypes.Structure):
    _fields_ = [("ptr", _vp * MAX_PEERS)]


class PeerSignalC(ctypes.Structure):
    _fields_ = [("pad", _vp * MAX_PEERS), ("counter", _vp), ("rank", _c_int), ("n", _c_int), ("timeout_ns", _c_ll)]


class RowsC(ctypes.Structure):
    _fields_ = [("ptr", _vp), ("ld", _c_ll), ("g_stride", _c_ll), ("lo_stride", _c_ll), ("hi_stride", _c_ll)]


class GemmDescC(ctypes.Structure):
    _fields_ = [("kind", _c_int), ("epi", _c_int), ("b_major", _c_int), ("groups", _c_int), ("nhi", _c_int),
                ("nlo", _c_int), ("seg_len", _c_int), ("M", _c_int), ("N", _c_int), ("K", _c_int),
                ("alpha", ctypes.c_float), ("pad_", _c_int), ("a", RowsC), ("b", RowsC), ("d", RowsC),
                ("aux", RowsC), ("fill", _vp)]


# name -> (restype, argtypes); mirrors include/parm_b200.h exactly.
SIGNATURES = {
    "parm_abi_version": (_c_int, []),
    "parm_last_error": (ctypes.c_char_p, []),
    "parm_gate_fwd": (_c_int, [_vp, _c_ll, _vp, _c_int, _c_int, _c_int, _c_int, _vp, _vp, _vp, _vp, _vp]),
    "parm_gate_counts_bytes": (_size, [_c_int, _c_int]),
    "parm_route_dispatch": (_c_int, [_vp, _c_ll, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_int, _vp, _vp, _vp, _c_int,
                                     _c_int, _vp, _c_ll, _c_ll, ctypes.POINTER(SlotViewC), ctypes.POINTER(IntFanC),
                                     _vp]),
    "parm_combine_fwd": (_c_int, [ctypes.POINTER(SlotViewC), _vp, _vp, _vp, _c_int, _c_int, _c_int, _vp, _c_ll,
                                  _vp]),
    "parm_combine_bwd_dispatch": (_c_int, [_vp, _c_ll, ctypes.POINTER(SlotViewC), _vp, _vp, _vp, _vp, _c_int,
                                           _c_int, _c_int, _c_int, _vp, _c_int, _c_int, _vp, _vp, _c_ll, _c_ll,
                                           ctypes.POINTER(SlotViewC), _vp]),
    "parm_dispatch_bwd": (_c_int, [ctypes.POINTER(SlotViewC), _vp, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int,
                                   _vp, _c_ll, _vp]),
    "parm_esp_sum": (_c_int, [ctypes.POINTER(SlotViewC), _c_int, _c_int, _c_int, _vp, _vp]),
    "parm_gate_wgrad_workspace": (_size, [_c_int, _c_int, _c_int]),
    "parm_gate_wgrad": (_c_int, [_vp, _c_ll, _vp, _c_int, _c_int, _c_int, _vp, _size, _vp, _c_int, _vp]),
    "parm_sum_chunks": (_c_int, [_vp, _c_int, _c_ll, _vp, _c_int, _vp]),
    "parm_gemm": (_c_int, [ctypes.POINTER(GemmDescC), _vp]),
    "parm_combine_fwd_fan": (_c_int, [ctypes.POINTER(SlotViewC), _vp, _vp, _vp, _c_int, _c_int, _c_int,
                                      ctypes.POINTER(RowFanC), _c_ll, _vp]),
    "parm_dispatch_bwd_fan": (_c_int, [ctypes.POINTER(SlotViewC), _vp, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int,
                                       ctypes.POINTER(RowFanC), _c_ll, _vp]),
    "parm_peer_barrier": (_c_int, [ctypes.POINTER(PeerSignalC), _c_int, _vp]),
    "parm_push_rows": (_c_int, [_vp, _c_int, _c_int, _c_int, _c_int, _vp, ctypes.POINTER(RowFanC), _vp]),
    "parm_fan_copy": (_c_int, [_vp, _c_ll, ctypes.POINTER(RowFanC), _vp]),
    "parm_gemm_peer": (_c_int, [ctypes.POINTER(GemmDescC), ctypes.POINTER(RowFanC), _c_ll, _c_ll, _vp]),
    "parm_gemm_multi_workspace": (ctypes.c_size_t, [ctypes.POINTER(GemmDescC), _c_int]),
    "parm_gemm_multi": (_c_int, [ctypes.POINTER(GemmDescC), _c_int, ctypes.POINTER(_c_int), _vp, ctypes.c_size_t,
                                 _c_int, ctypes.POINTER(RowFanC), _c_ll, _c_ll, _vp]),
}

ABI_VERSION = 16


class ParmError(RuntimeError):
    """A C-ABI call returned a non-zero status."""


class ParmArgError(ParmError, ValueError):
    """Status 1: argument validation failed inside the library."""


_lib = None


def load(path: str | os.PathLike | None = None) -> ctypes.CDLL:
    """Load (once) and type the library; raise loudly when it is absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path is not None else LIB_PATH
    if not p.exists():
        raise ImportError(
            f"{p} is missing: build it with `python -m paper_2407_00599_b200.build` (or __graft_entry__.build()); "
            "there is no CPU fallback for the Parm MoE kernels")
    lib = ctypes.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.parm_abi_version() != ABI_VERSION:
        raise ImportError(f"{p}: ABI version {lib.parm_abi_version()} != {ABI_VERSION}")
    if path is None:
        _lib = lib
    return lib


# Kernel launches each entry point issues on success when not 1 (bench.py's gpu_launches).
# (parm_gate_wgrad: 1 -- the partial sum runs in the same cooperative launch whenever its CTAs
# fit on the SMs at once, true up to M = 4096 at E <= 8; wider launches add a second kernel.)
LAUNCHES_PER_CALL: dict = {}
launch_count = 0


def call(name: str, *args) -> None:
    global launch_count
    lib = load()
    rc = getattr(lib, name)(*args)
    launch_count += LAUNCHES_PER_CALL.get(name, 1)
    if rc != 0:
        msg = lib.parm_last_error().decode(errors="replace")
        if rc == 1:
            raise ParmArgError(msg)
        raise ParmError(f"{name} failed ({rc}): {msg}")
