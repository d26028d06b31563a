"""B200-native GraphGuess engine (arXiv 2104.10039): the approximate
pull-gather hot path as sm_100a CUDA behind the reference's plugin API.

Importing loads libggb.so and checks every C-ABI symbol; a missing or
broken extension raises ImportError (no CPU fallback)."""
from ._lib import lib as _load

_load()

from .engine import (  # noqa: E402
    DeviceBuffer, DeviceView, Exchange, bp_priors,
    BeliefPropagationProgram, DeviceGraph, EdgeBeliefPropagationProgram, EngineConfig, EngineError,
    ErrorReport, GgbError, Graph, IterationMode, IterationRecord, PageRankProgram, RunReport,
    Scheme, SsspProgram, WccProgram, bp_spec, mode_for, pagerank_spec, partition_plan,
    relative_error, run, scheme_from_name, select_superstep_iterations, sparsify, sssp_spec,
    stretch_error, topk_error, unpack_bitmap, validate, wcc_spec,
)

__all__ = [
    "DeviceBuffer", "DeviceView", "Exchange", "bp_priors", "BeliefPropagationProgram", "DeviceGraph", "EdgeBeliefPropagationProgram", "EngineConfig",
    "EngineError", "ErrorReport", "GgbError", "Graph", "IterationMode", "IterationRecord",
    "PageRankProgram", "RunReport", "Scheme", "SsspProgram", "WccProgram", "bp_spec", "mode_for",
    "pagerank_spec", "partition_plan", "relative_error", "run", "scheme_from_name",
    "select_superstep_iterations", "sparsify", "sssp_spec", "stretch_error", "topk_error",
    "unpack_bitmap", "validate", "wcc_spec",
]
