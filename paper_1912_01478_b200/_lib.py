"""ctypes binding of libhcb.so (include/hcb.h).

There is exactly one compute path: the in-tree CUDA library.  If it is missing
or no CUDA device is visible, every entry point raises -- there is no CPU
fallback (the reference's `auto` backend silently falls back to numpy,
_backend.py:28-31; this package deliberately does not).
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import torch

PKG = Path(__file__).resolve().parent
# HCB_LIB selects an alternative in-tree build (tuning experiments only)
LIB_PATH = PKG / os.environ.get("HCB_LIB", "libhcb.so")

HC_OK = 0
HC_ERR_INVALID = -1
HC_ERR_CUDA = -2
HC_ERR_WL_OVERFLOW = -3
HC_ERR_WORKSPACE = -4
HC_ERR_UNCOLORED = -5
HC_ERR_DUPLICATE = -6
HC_ERR_RECORDS = -7
HC_ERR_TIMEOUT = -8
HC_ERR_STALLED = -9

MODE_CODES = {"data": 0, "topo": 1, "hybrid": 2}


class HcError(RuntimeError):
    """A libhcb call failed; `code` is the HC_ERR_* value."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"libhcb error {code}: {msg}")
        self.code = code


class RoundRec(ctypes.Structure):
    """hc_round_rec (include/hcb.h) == RoundRecord fields (driver.py:47-54)."""

    _fields_ = [
        ("round", ctypes.c_int64),
        ("topo", ctypes.c_int64),
        ("wl_in", ctypes.c_int64),
        ("wl_out", ctypes.c_int64),
        ("conflicts", ctypes.c_int64),
        ("ns", ctypes.c_int64),
    ]


REC_FIELDS = 6  # int64 words per hc_round_rec


class SolvePlan(ctypes.Structure):
    """hc_solve_plan (include/hcb.h): the per-graph kernel choice of a planned workspace."""

    _fields_ = [("num_nodes", ctypes.c_int64), ("num_edges", ctypes.c_int64),
                ("narrow", ctypes.c_int32), ("x16", ctypes.c_int32), ("c16", ctypes.c_int32),
                ("small", ctypes.c_int32), ("ell", ctypes.c_int32), ("live", ctypes.c_int32),
                ("totals_offset", ctypes.c_int64), ("reserved", ctypes.c_int64 * 3)]

_lib = None

_i64 = ctypes.c_int64
_p = ctypes.c_void_p
_SIGS = {
    "hc_last_error": (ctypes.c_char_p, []),
    "hc_version": (ctypes.c_int, []),
    "hc_device_info": (ctypes.c_int, [_p, _p]),
    "hc_k_assign_from_list": (ctypes.c_int, [_p, _p, _p, _p, _p, _p, _i64, _i64, _i64, _p]),
    "hc_k_assign_sweep": (ctypes.c_int, [_p, _p, _p, _p, _p, _i64, _i64, _i64, _p, _p, _p]),
    "hc_k_resolve_from_list": (ctypes.c_int, [_p, _p, _p, _p, _p, _p, _i64, _i64, _p, _i64, _p, _p, _p, _p]),
    "hc_k_resolve_sweep": (ctypes.c_int, [_p, _p, _p, _p, _p, _i64, _i64, _p, _i64, _p, _p, _p, _p]),
    "hc_k_bench_from_list": (ctypes.c_int, [_p, _i64, _p, _i64, _p, _i64, _p, _p]),
    "hc_k_bench_sweep": (ctypes.c_int, [_p, _i64, _i64, _p, _i64, _p, _p]),
    "hc_k_commit_list": (ctypes.c_int, [_p, _p, _p, _i64, _p]),
    "hc_k_commit_stamped": (ctypes.c_int, [_p, _p, _p, _i64, _i64, _p]),
    "hc_wl_sort_workspace_bytes": (ctypes.c_size_t, [_i64]),
    "hc_wl_swap_and_sort": (ctypes.c_int, [_p, _p, _i64, _p, _p, _p, ctypes.c_size_t, _p]),
    "hc_solve_workspace_bytes": (ctypes.c_size_t, [_i64, _i64]),
    "hc_solve_set_formats": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    "hc_solve_set_small": (ctypes.c_int, [ctypes.c_int]),
    "hc_solve_set_l2_window": (ctypes.c_int, [ctypes.c_int]),
    "hc_solve_set_ell": (ctypes.c_int, [ctypes.c_int]),
    "hc_solve_set_x8": (ctypes.c_int, [ctypes.c_int]),
    "hc_solve_set_live": (ctypes.c_int, [ctypes.c_int]),
    "hc_solve": (ctypes.c_int, [_p, _p, _i64, _i64, ctypes.c_int, _i64, _p, _p, _i64, _p, _p, ctypes.c_size_t, _p]),
    "hc_solve_plain": (ctypes.c_int, [_p, _p, _i64, _i64, ctypes.c_int, _i64, _p, _p, _i64, _p, _p, ctypes.c_size_t, _p]),
    "hc_solve_plan_graph": (ctypes.c_int, [_p, _p, _i64, _i64, _p, ctypes.c_size_t, _p, _p]),
    "hc_solve_launch": (ctypes.c_int, [_p, _p, _p, ctypes.c_int, _i64, _p, _p, _i64, _p, _p, ctypes.c_size_t, _p]),
    "hc_solve_stats": (ctypes.c_int, [_p, _p, _i64, _i64, ctypes.c_int, _i64, _p, _p, _i64, _p, _p, _p, ctypes.c_size_t, _p]),
    "hc_mg_shared_bytes": (ctypes.c_size_t, [_i64]),
    "hc_mg_workspace_bytes": (ctypes.c_size_t, [_i64, _i64, _i64, _i64]),
    "hc_mg_alloc_shared": (ctypes.c_int, [ctypes.c_size_t, _p]),
    "hc_mg_free_shared": (ctypes.c_int, [_p]),
    "hc_mg_ipc_export": (ctypes.c_int, [_p, _p, _p]),
    "hc_mg_ipc_import": (ctypes.c_int, [_p, _i64, _p]),
    "hc_mg_ipc_close": (ctypes.c_int, [_p, _i64]),
    "hc_mg_solve": (ctypes.c_int, [_p, _p, _i64, _i64, _p, ctypes.c_int, ctypes.c_int, _p, ctypes.c_int,
                                   _i64, _p, _p, _i64, ctypes.c_int, _i64, _i64, _p, ctypes.c_size_t, _p]),
    "hc_mg_wait": (ctypes.c_int, [_p, _p, _p]),
    "hc_mg_set_exchange": (ctypes.c_int, [ctypes.c_int]),
    "hc_mg_prepare": (ctypes.c_int, [_p, _p, _i64, _i64, _p, ctypes.c_int, ctypes.c_int, _p, ctypes.c_int,
                                     _i64, _p, _p, _i64, ctypes.c_int, _i64, _i64, _p, ctypes.c_size_t, _p]),
    "hc_mg_launch": (ctypes.c_int, [_p, _p]),
    "hc_dist_boundary": (ctypes.c_int, [_p, _p, _i64, _i64, _p, _p]),
    "hc_dist_assign": (ctypes.c_int, [_p, _p, _p, _p, _i64, _i64, _p, _p, _p, _p, _p]),
    "hc_dist_resolve": (ctypes.c_int, [_p, _p, _p, _p, _i64, _i64, _p, _p, _p, _p, _p, _p, _p, _p]),
    "hc_dist_apply": (ctypes.c_int, [_p, _p, _p, _i64, _p]),
    "hc_dist_colors": (ctypes.c_int, [_p, _i64, _i64, _p, _p]),
    "hc_push_bench_workspace_bytes": (ctypes.c_size_t, [_i64]),
    "hc_push_bench": (ctypes.c_int, [_i64, _i64, ctypes.c_int, _p, _p, _p, _i64, _p, _p, ctypes.c_size_t, _p]),
    "hc_build_csr_workspace_bytes": (ctypes.c_size_t, [_i64, _i64]),
    "hc_build_csr": (ctypes.c_int, [_p, _i64, _i64, _p, _p, _p, _p, ctypes.c_size_t, _p]),
    "hc_build_csr_rows_workspace_bytes": (ctypes.c_size_t, [_i64, _i64, _i64, _i64]),
    "hc_build_csr_rows": (ctypes.c_int, [_p, _i64, _i64, _i64, _i64, _i64, _p, _p, _p, _p, ctypes.c_size_t, _p]),
    "hc_edge_degrees": (ctypes.c_int, [_p, _i64, _i64, _p, _p]),
    "hc_verify_rows": (ctypes.c_int, [_p, _p, _i64, _i64, _p, _p, _p, _p]),
    "hc_gen_grid": (ctypes.c_int, [_i64, _i64, _p, _p]),
    "hc_gen_er": (ctypes.c_int, [_i64, _i64, ctypes.c_uint64, _p, _p]),
    "hc_gen_rmat": (ctypes.c_int, [ctypes.c_int, _i64, ctypes.c_uint64, _p, _p]),
    "hc_verify": (ctypes.c_int, [_p, _p, _i64, _p, _p, _p, _p]),
    "hc_colors_used": (ctypes.c_int, [_p, _i64, _p, _p, _p]),
    "hc_narrow_i64_i32": (ctypes.c_int, [_p, _p, _i64, _p]),
    "hc_csr_check_lower_first": (ctypes.c_int, [_p, _p, _i64, _p, _p, _p]),
    "hc_csr_partition_lower_first": (ctypes.c_int, [_p, _p, _p, _i64, _p]),
    "hc_mtx_workspace_bytes": (ctypes.c_size_t, [_i64]),
    "hc_mtx_parse": (ctypes.c_int, [_p, _i64, ctypes.c_int, _i64, _i64, _i64, _p, _p, _p, _p, _p, _p, _p,
                                    ctypes.c_size_t, _p]),
    "hc_degree_stats_workspace_bytes": (ctypes.c_size_t, []),
    "hc_degree_stats": (ctypes.c_int, [_p, _i64, _p, _p, _p, _p, ctypes.c_size_t, _p]),
}

EXPORTED_SYMBOLS = tuple(_SIGS)


def load():
    """Load libhcb.so (raises if it was not built; see __graft_entry__.build)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `make -C {PKG / 'csrc'}` "
                "(or __graft_entry__.build()); there is no CPU fallback"
            )
        L = ctypes.CDLL(str(LIB_PATH))
        variant = "HCB_LIB" in os.environ  # tuning builds may predate newer entry points
        for name, (res, args) in _SIGS.items():
            if variant and not hasattr(L, name):
                continue
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def device() -> torch.device:
    """The CUDA device every call runs on; raises when none is visible."""
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device visible: the IPGC hot path runs on the GPU only")
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def check(rc: int) -> None:
    if rc != HC_OK:
        msg = load().hc_last_error().decode(errors="replace")
        if rc == HC_ERR_INVALID:
            raise ValueError(msg)
        if rc == HC_ERR_DUPLICATE:
            raise AssertionError(msg)  # worklist.py:85-88
        raise HcError(rc, msg)


def ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    return t.data_ptr() if t.numel() else None


def workspace(nbytes: int, dev: torch.device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=dev)


if os.environ.get("HCB_EAGER_LOAD") == "1":  # pragma: no cover
    load()
