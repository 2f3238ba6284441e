"""ctypes binding of libleanot_b200.so (include/leanot_b200.h).

The shared library is built in-tree by `make` (see __graft_entry__.build()).
There is no fallback: if the library or a CUDA device is missing, every entry
point raises.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("LEANOT_LIB", str(_HERE / "libleanot_b200.so")))

LEANOT_OK = 0
LEANOT_EINVAL = -1
MAX_K = 16
COST_STORED, COST_POINTS, COST_GRID = 0, 1, 2


class CostT(C.Structure):
    _fields_ = [("kind", C.c_int32), ("p", C.c_int32), ("dim", C.c_int32), ("height", C.c_int32),
                ("width", C.c_int32), ("_pad", C.c_int32), ("n", C.c_int64), ("ld", C.c_int64),
                ("row_base", C.c_int64), ("mat", C.c_void_p), ("feat", C.c_void_p),
                ("grid_coords", C.c_void_p), ("inv_scale", C.c_double), ("sup_norm", C.c_double),
                ("norms", C.c_void_p)]


class WsetsT(C.Structure):
    _fields_ = [("K", C.c_int32), ("_pad", C.c_int32), ("a", C.c_void_p), ("b", C.c_void_p * MAX_K)]


class ParamsT(C.Structure):
    _fields_ = [("eta", C.c_double), ("eta_mu", C.c_double), ("tau_p", C.c_double),
                ("tau_mu", C.c_double), ("beta", C.c_double), ("alpha", C.c_double)]


class DxgPlanT(C.Structure):
    _fields_ = [("cost", CostT), ("prm", ParamsT), ("n", C.c_int64), ("row0", C.c_int64),
                ("row1", C.c_int64), ("splits", C.c_int32), ("nblk_upd", C.c_int32)] + [
        (name, C.c_void_p) for name in (
            "r", "c", "c_tilde", "delta", "b", "b_bar", "bprime", "sd", "scal", "shift", "m", "S",
            "coef", "rowstat", "slab", "col", "partial", "evalbuf", "flags", "beta")]


class BaryPlanT(C.Structure):
    _fields_ = [("cost", CostT), ("prm", ParamsT), ("n", C.c_int64), ("row0", C.c_int64), ("row1", C.c_int64),
                ("ns", C.c_int64), ("m", C.c_int32), ("splits", C.c_int32), ("nblk_upd", C.c_int32), ("_pad", C.c_int32)] + [
        (name, C.c_void_p) for name in (
            "w", "c", "c_tilde", "delta", "b", "b_bar", "bprime", "sd", "scal", "shift", "mu", "S", "L", "r",
            "coef", "rowstat", "slab", "col", "partial", "scratch", "evalbuf", "flags")]


_lib = None


def lib():
    """Load the library once; raise loudly if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()); "
                           "there is no CPU fallback")
    L = C.CDLL(str(LIB_PATH))
    vp, i64, i32, dbl = C.c_void_p, C.c_int64, C.c_int32, C.c_double
    sigs = {
        "leanot_version": ([], C.c_int),
        "leanot_last_error": ([], C.c_char_p),
        "leanot_device_sm_count": ([C.c_int, C.POINTER(C.c_int)], C.c_int),
        "leanot_dxg_default_splits": ([i64, i64, C.POINTER(C.c_int)], C.c_int),
        "leanot_cost_block": ([C.POINTER(CostT), i64, i64, vp, i64, vp], C.c_int),
        "leanot_stored_max": ([vp, i64, i64, i64, vp, vp, vp], C.c_int),
        "leanot_stored_normalize": ([vp, i64, i64, i64, dbl, vp], C.c_int),
        "leanot_points_sup": ([vp, i64, C.c_int, C.c_int, vp, vp, vp], C.c_int),
        "leanot_points_norms": ([vp, i64, C.c_int, vp, vp], C.c_int),
        "leanot_sum_partials": ([vp, C.c_int, i64, vp, vp], C.c_int),
        "leanot_dxg_iterate_eval": ([C.POINTER(DxgPlanT), C.c_int, C.c_int, vp], C.c_int),
        "leanot_bary_rows": ([C.POINTER(BaryPlanT), C.c_int, vp, vp], C.c_int),
        "leanot_bary_rnorm": ([C.POINTER(BaryPlanT), vp, vp, vp], C.c_int),
        "leanot_bary_cols": ([C.POINTER(BaryPlanT), vp, vp], C.c_int),
        "leanot_hash_fill": ([vp, i64, i64, i64, i64, C.c_uint64, vp], C.c_int),
        "leanot_sweep_ws_doubles": ([i64, i64, C.c_int], i64),
        "leanot_column_marginals": ([C.POINTER(CostT), i64, i64, C.POINTER(WsetsT), vp, vp, vp, vp], C.c_int),
        "leanot_row_lse": ([C.POINTER(CostT), i64, i64, C.POINTER(WsetsT), vp, vp, vp], C.c_int),
        "leanot_plan_stats": ([C.POINTER(CostT), i64, i64, C.POINTER(WsetsT), vp, vp, vp, vp, vp], C.c_int),
        "leanot_row_min": ([C.POINTER(CostT), i64, i64, vp, vp, vp], C.c_int),
        "leanot_row_lse_affine": ([C.POINTER(CostT), i64, i64, vp, dbl, dbl, vp, vp], C.c_int),
        "leanot_dxg_prepare": ([C.POINTER(DxgPlanT), dbl, dbl, dbl, C.c_int, vp], C.c_int),
        "leanot_dxg_sweep": ([C.POINTER(DxgPlanT), C.c_int, vp], C.c_int),
        "leanot_debug_sr_trace": ([vp], C.c_int),
        "leanot_dxg_update": ([C.POINTER(DxgPlanT), vp], C.c_int),
        "leanot_dxg_eval": ([C.POINTER(DxgPlanT), vp], C.c_int),
        "leanot_dxg_iterate": ([C.POINTER(DxgPlanT), C.c_int, vp], C.c_int),
        "leanot_graph_create": ([C.POINTER(DxgPlanT), C.c_int, C.POINTER(vp), vp], C.c_int),
        "leanot_graph_launch": ([vp, vp], C.c_int),
        "leanot_graph_destroy": ([vp], C.c_int),
        "leanot_bary_rmap": ([vp, C.c_int, i64, vp, vp, vp, vp], C.c_int),
        "leanot_sync": ([vp], C.c_int),
        "leanot_bary_prepare": ([C.POINTER(BaryPlanT), dbl, dbl, dbl, C.c_int, vp], C.c_int),
        "leanot_bary_sweep": ([C.POINTER(BaryPlanT), C.c_int, vp], C.c_int),
        "leanot_bary_update": ([C.POINTER(BaryPlanT), vp], C.c_int),
        "leanot_bary_eval": ([C.POINTER(BaryPlanT), vp], C.c_int),
        "leanot_col_lse_ws_doubles": ([i64, i64], i64),
        "leanot_col_lse": ([C.POINTER(CostT), i64, i64, vp, dbl, vp, vp, vp], C.c_int),
        "leanot_eta_log_minus": ([vp, vp, dbl, i64, vp, vp], C.c_int),
        "leanot_sinkhorn_psi": ([vp, vp, vp, dbl, i64, vp, vp, vp], C.c_int),
        "leanot_eot_dual": ([vp, vp, vp, vp, vp, dbl, i64, vp, vp], C.c_int),
        "leanot_sinkhorn_colmarg": ([vp, vp, dbl, i64, vp, vp], C.c_int),
        "leanot_ibp_rows": ([vp, C.c_int, i64, dbl, vp, vp, vp, vp], C.c_int),
        "leanot_materialize_plan": ([C.POINTER(CostT), dbl, vp, vp, vp, vp, i64, vp], C.c_int),
        "leanot_round_polytope": ([vp, i64, i64, vp, vp, vp, vp], C.c_int),
        "leanot_plan_cost": ([C.POINTER(CostT), vp, i64, vp, vp, vp], C.c_int),
        "leanot_pdxg_rows": ([C.POINTER(CostT), vp, i64, dbl, dbl, dbl, vp, vp, vp], C.c_int),
        "leanot_pdxg_colsum": ([vp, i64, i64, vp, vp, vp], C.c_int),
        "leanot_grid_sep_ws_doubles": ([C.POINTER(CostT)], i64),
        "leanot_grid_sep_lse": ([C.POINTER(CostT), vp, vp, vp, vp, vp], C.c_int),
        "leanot_grid_sep_colsum": ([C.POINTER(CostT), vp, vp, vp, vp, vp, vp], C.c_int),
        "leanot_grid_sep_lse_eta_ws_doubles": ([C.POINTER(CostT), C.c_int], i64),
        "leanot_grid_sep_lse_eta": ([C.POINTER(CostT), vp, C.c_int, i64, C.c_double, vp, i64, vp, vp], C.c_int),
    }
    for name, (args, res) in sigs.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


EXPORTS = (
    "leanot_version", "leanot_last_error", "leanot_device_sm_count", "leanot_dxg_default_splits",
    "leanot_cost_block", "leanot_stored_max", "leanot_stored_normalize", "leanot_points_sup", "leanot_points_norms", "leanot_sum_partials",
    "leanot_bary_rows", "leanot_bary_rnorm", "leanot_bary_cols", "leanot_dxg_iterate_eval",
    "leanot_hash_fill", "leanot_sweep_ws_doubles", "leanot_column_marginals", "leanot_row_lse",
    "leanot_plan_stats", "leanot_row_min", "leanot_row_lse_affine", "leanot_dxg_prepare",
    "leanot_dxg_sweep", "leanot_debug_sr_trace", "leanot_dxg_update", "leanot_dxg_eval", "leanot_dxg_iterate",
    "leanot_graph_create", "leanot_graph_launch", "leanot_graph_destroy", "leanot_bary_rmap",
    "leanot_sync", "leanot_bary_prepare", "leanot_bary_sweep", "leanot_bary_update", "leanot_bary_eval",
    "leanot_col_lse_ws_doubles", "leanot_col_lse", "leanot_eta_log_minus", "leanot_sinkhorn_psi", "leanot_eot_dual",
    "leanot_sinkhorn_colmarg", "leanot_ibp_rows", "leanot_materialize_plan", "leanot_round_polytope",
    "leanot_plan_cost", "leanot_pdxg_rows", "leanot_pdxg_colsum", "leanot_grid_sep_ws_doubles", "leanot_grid_sep_lse", "leanot_grid_sep_colsum", "leanot_grid_sep_lse_eta", "leanot_grid_sep_lse_eta_ws_doubles",
)


def check(rc: int, what: str = "") -> None:
    """Map a status code to the reference's exception types (ValueError for bad input)."""
    if rc == LEANOT_OK:
        return
    msg = lib().leanot_last_error().decode(errors="replace")
    if rc == LEANOT_EINVAL:
        raise ValueError(msg or what)
    raise RuntimeError(f"{what}: {msg}")


def ptr(t) -> int:
    """Device pointer of a torch tensor (or None)."""
    return None if t is None else t.data_ptr()


def stream_handle(torch_stream=None):
    import torch
    s = torch_stream if torch_stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2511_11359_b200 needs a CUDA device (B200, sm_100a); no CPU fallback exists")
    lib()


def env_device():
    import torch
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return torch.device("cuda", local % max(1, torch.cuda.device_count()))
