"""ctypes binding of libggb.so (include/ggb.h). Loading fails loudly: there
is no CPU fallback anywhere in this package."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GGB_LIB_PATH", os.path.join(HERE, "libggb.so"))  # override: A/B builds

GG_OK, GG_INVALID_ARGUMENT, GG_INVALID_PROPERTY, GG_CUDA, GG_NCCL, GG_OOM, GG_INTERNAL = range(7)
GG_W_NONE, GG_W_U32, GG_W_F32, GG_W_F64 = range(4)

# every symbol include/ggb.h declares (checked at load and by tests)
EXPORTS = (
    "gg_status_string", "gg_abi_version", "gg_bp_priors_device", "gg_device_upload",
    "gg_device_free", "gg_device_copy", "gg_last_projection", "gg_topk_error_dev",
    "gg_relative_error_dev", "gg_stretch_error_dev", "gg_dev_graph_load", "gg_dev_graph_save",
    "gg_dev_graph_weight_kind", "gg_dev_graph_create", "gg_dev_graph_create_for_run",
    "gg_dev_graph_destroy",
    "gg_dev_graph_info", "gg_dev_graph_create_rmat", "gg_dev_graph_export", "gg_bp_priors",
    "gg_run_pr", "gg_run_sssp", "gg_run_wcc", "gg_run_bp", "gg_validate", "gg_mode_for",
    "gg_select_superstep_iterations", "gg_sparsify", "gg_partition_plan", "gg_nccl_unique_id",
    "gg_exchange_nccl_create", "gg_exchange_local_group", "gg_exchange_destroy", "gg_exchange_set_fused", "gg_exchange_selftest", "gg_topk_error", "gg_relative_error",
    "gg_stretch_error", "gg_dev_graph_symmetrized",
)


class CscView(C.Structure):
    _fields_ = [("n", C.c_uint64), ("e", C.c_uint64), ("offsets", C.c_void_p),
                ("sources", C.c_void_p), ("weight_kind", C.c_int), ("weights", C.c_void_p),
                ("out_degree", C.c_void_p)]


class PartOpts(C.Structure):
    _fields_ = [("device", C.c_int), ("rank", C.c_int), ("nranks", C.c_int),
                ("exchange", C.c_void_p)]


class EngineConfigC(C.Structure):
    _fields_ = [("scheme", C.c_int32), ("sigma", C.c_double), ("theta", C.c_double),
                ("alpha", C.c_uint64), ("max_iterations", C.c_uint64), ("seed", C.c_uint64),
                ("threads", C.c_uint32)]


class IterRecordC(C.Structure):
    _fields_ = [("mode", C.c_int32), ("processed_edges", C.c_uint64),
                ("active_vertices", C.c_uint64), ("wall_seconds", C.c_double),
                ("kernel_ms", C.c_double), ("rebuild_ms", C.c_double),
                ("exchange_ms", C.c_double), ("algo_bytes", C.c_uint64),
                ("edge_ms", C.c_double), ("vertex_ms", C.c_double),
                ("edge_bytes", C.c_uint64), ("vertex_bytes", C.c_uint64)]


class RunSummaryC(C.Structure):
    _fields_ = [("iterations_run", C.c_uint64), ("total_processed_edges", C.c_uint64),
                ("total_wall_seconds", C.c_double), ("kept_edges", C.c_uint64),
                ("kernel_launches", C.c_uint32), ("exchange_fused", C.c_uint32)]


class ErrorC(C.Structure):
    _fields_ = [("iteration", C.c_uint64), ("vertex", C.c_uint32), ("msg", C.c_char * 256)]


ABI_VERSION = 5  # include/ggb.h GGB_ABI_VERSION


class RunOptsC(C.Structure):
    _fields_ = [("out_flags", C.c_void_p), ("timing", C.c_int), ("device_output", C.c_int),
                ("grid_ctas", C.c_uint32)]


class PrParams(C.Structure):
    _fields_ = [("damping", C.c_double), ("epsilon", C.c_double)]


class SsspParams(C.Structure):
    _fields_ = [("source", C.c_uint32), ("graded", C.c_int32)]


class BpParams(C.Structure):
    _fields_ = [("states", C.c_int32), ("coupling", C.c_double), ("epsilon", C.c_double),
                ("prior_table", C.c_void_p), ("prior_on_device", C.c_int32)]


class RmatParams(C.Structure):
    _fields_ = [("scale", C.c_uint32), ("edge_factor", C.c_uint32), ("seed", C.c_uint64),
                ("a", C.c_double), ("b", C.c_double), ("c", C.c_double),
                ("symmetrize", C.c_int32), ("weight_kind", C.c_int)]


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libggb.so not found at {LIB_PATH}: run __graft_entry__.build() (no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    missing = [s for s in EXPORTS if not hasattr(L, s)]
    # an A/B library (GGB_LIB_PATH, tools/ab.py) may predate newer entry points
    if missing and not os.environ.get("GGB_LIB_PATH"):
        raise ImportError(f"libggb.so lacks symbols {missing}")
    L.gg_abi_version.restype = C.c_int
    if L.gg_abi_version() != ABI_VERSION:
        raise ImportError(f"libggb.so ABI {L.gg_abi_version()} != {ABI_VERSION} (stale build: "
                          "run __graft_entry__.build())")
    P = C.POINTER
    vp = C.c_void_p
    L.gg_status_string.argtypes = [C.c_int]
    L.gg_status_string.restype = C.c_char_p
    L.gg_dev_graph_create.argtypes = [P(CscView), P(PartOpts), P(vp), P(ErrorC)]
    L.gg_dev_graph_create_for_run.argtypes = [P(CscView), P(PartOpts), C.c_double, C.c_uint64,
                                              P(vp), P(ErrorC)]
    L.gg_dev_graph_create_rmat.argtypes = [P(RmatParams), P(PartOpts), P(vp), P(ErrorC)]
    L.gg_dev_graph_destroy.argtypes = [vp]
    L.gg_dev_graph_info.argtypes = [vp] + [P(C.c_uint64)] * 5
    L.gg_dev_graph_export.argtypes = [vp, vp, vp, vp, vp]
    L.gg_dev_graph_symmetrized.argtypes = [vp, vp, P(vp), P(ErrorC)]
    L.gg_bp_priors.argtypes = [C.c_uint64, C.c_uint64, vp]
    common = [P(IterRecordC), C.c_uint64, P(RunSummaryC), P(RunOptsC), P(ErrorC)]
    L.gg_run_pr.argtypes = [vp, P(EngineConfigC), P(PrParams), vp] + common
    L.gg_run_sssp.argtypes = [vp, P(EngineConfigC), P(SsspParams), vp] + common
    L.gg_run_wcc.argtypes = [vp, P(EngineConfigC), vp] + common
    L.gg_run_bp.argtypes = [vp, P(EngineConfigC), P(BpParams), vp] + common
    L.gg_bp_priors_device.argtypes = [C.c_uint64, C.c_uint64, P(vp)]
    L.gg_device_upload.argtypes = [vp, C.c_uint64, P(vp)]
    L.gg_device_free.argtypes = [vp]
    L.gg_device_copy.argtypes = [vp, C.c_uint64, P(vp)]
    L.gg_dev_graph_load.argtypes = [C.c_char_p, P(PartOpts), P(vp), P(ErrorC)]
    L.gg_dev_graph_save.argtypes = [vp, C.c_char_p, P(ErrorC)]
    L.gg_dev_graph_weight_kind.argtypes = [vp]
    L.gg_dev_graph_weight_kind.restype = C.c_int32
    L.gg_last_projection.argtypes = [vp, P(vp)]
    L.gg_topk_error_dev.argtypes = [vp, vp, C.c_uint64, C.c_uint64, P(C.c_double)]
    L.gg_relative_error_dev.argtypes = [vp, vp, C.c_uint64, P(C.c_double)]
    L.gg_stretch_error_dev.argtypes = [vp, vp, C.c_uint64, P(C.c_double), P(ErrorC)]
    L.gg_validate.argtypes = [P(EngineConfigC), P(ErrorC)]
    L.gg_mode_for.argtypes = [C.c_int32, C.c_uint64, C.c_uint64]
    L.gg_mode_for.restype = C.c_int32
    L.gg_select_superstep_iterations.argtypes = [C.c_uint64, C.c_uint64, C.c_int32, vp, C.c_uint64]
    L.gg_select_superstep_iterations.restype = C.c_uint64
    L.gg_sparsify.argtypes = [C.c_uint64, C.c_double, C.c_uint64, vp, P(ErrorC)]
    L.gg_partition_plan.argtypes = [C.c_uint64, vp, C.c_int, vp]
    L.gg_nccl_unique_id.argtypes = [vp]
    L.gg_exchange_nccl_create.argtypes = [vp, C.c_int, C.c_int, P(vp), P(ErrorC)]
    L.gg_exchange_destroy.argtypes = [vp]
    L.gg_exchange_selftest.argtypes = [vp, P(ErrorC)]
    if hasattr(L, "gg_exchange_set_fused"):
        L.gg_exchange_set_fused.argtypes = [vp, C.c_int]
    L.gg_exchange_local_group.argtypes = [C.c_int, P(vp)]
    L.gg_topk_error.argtypes = [vp, vp, C.c_uint64, C.c_uint64, P(C.c_double)]
    L.gg_relative_error.argtypes = [vp, vp, C.c_uint64, P(C.c_double)]
    L.gg_stretch_error.argtypes = [vp, vp, C.c_uint64, P(C.c_double)]
    for s in EXPORTS:
        if s not in ("gg_status_string", "gg_mode_for", "gg_select_superstep_iterations",
                     "gg_abi_version") and s not in missing:
            getattr(L, s).restype = C.c_int
    _lib = L
    return L


def status_string(code: int) -> str:
    return lib().gg_status_string(code).decode()
