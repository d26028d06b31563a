"""Host-side mirror of the reference's operator API for the hot path.

Same names, argument meaning and error behaviour as the reference
(/root/reference/proj/core/include/gg/*.hpp):

  Graph (graph.hpp:29-49), EngineConfig (engine.hpp:28-36), Scheme /
  IterationMode (:19, :24), IterationRecord / RunReport (:42-56),
  EngineError (:60-74), run (:141-249), sparsify (:97), mode_for (:106),
  select_superstep_iterations (:101-103), validate (:40), the program types
  and factories of algorithms.hpp, and the metrics of metrics.hpp.

Every compute call goes through libggb.so (include/ggb.h); errors map
std::invalid_argument -> ValueError and gg::EngineError -> EngineError.
"""
from __future__ import annotations

import ctypes as C
import os
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L


class Scheme(enum.IntEnum):
    accurate = 0
    sp = 1
    sms = 2
    gg = 3


class IterationMode(enum.IntEnum):
    approximate = 0
    accurate = 1
    superstep = 2


def scheme_from_name(name: str) -> Scheme:  # engine.cpp:29-35
    try:
        return Scheme[name]
    except KeyError:
        raise ValueError(f"unknown scheme: {name}") from None


class EngineError(RuntimeError):
    """gg::EngineError (engine.hpp:60-74): invalid property at (iteration, vertex)."""

    def __init__(self, iteration: int, vertex: int):
        super().__init__(f"invalid property at iteration {iteration}, vertex {vertex}")
        self.iteration = iteration
        self.vertex = vertex


class GgbError(RuntimeError):
    """CUDA / NCCL / OOM / internal failures of the device engine."""


def _raise(code: int, err: L.ErrorC | None):
    if code == L.GG_OK:
        return
    msg = err.msg.decode() if err is not None else L.status_string(code)
    if code == L.GG_INVALID_ARGUMENT:
        raise ValueError(msg)
    if code == L.GG_INVALID_PROPERTY:
        raise EngineError(int(err.iteration), int(err.vertex))
    raise GgbError(f"{L.status_string(code)}: {msg}")


# --------------------------------------------------------------------------
# Graph
# --------------------------------------------------------------------------
class Graph:
    """Pull CSC (graph.hpp:29-49). in_offsets u64[N+1], in_sources u32[E],
    weights (None or per-edge array: uint32 / float32 / float64), out_degree."""

    def __init__(self, n, in_offsets, in_sources, weights=None, out_degree=None):
        self.n = int(n)
        self.in_offsets = np.ascontiguousarray(in_offsets, dtype=np.uint64)
        self.in_sources = np.ascontiguousarray(in_sources, dtype=np.uint32)
        if self.in_offsets.shape[0] != self.n + 1:
            raise ValueError("graph: offset array has wrong length")
        if weights is not None:
            weights = np.ascontiguousarray(weights)
            if weights.dtype not in (np.uint32, np.float32, np.float64):
                weights = weights.astype(np.float64)
        self.weights = weights
        if out_degree is None:
            out_degree = (np.bincount(self.in_sources, minlength=self.n).astype(np.uint32)
                          if self.n else np.zeros(0, np.uint32))
        self.out_degree = np.ascontiguousarray(out_degree, dtype=np.uint32)

    def num_vertices(self) -> int:
        return self.n

    def num_edges(self) -> int:
        return int(self.in_sources.shape[0])

    def weighted(self) -> bool:
        return self.weights is not None

    def weight_kind(self) -> int:
        if self.weights is None:
            return L.GG_W_NONE
        return {np.dtype(np.uint32): L.GG_W_U32, np.dtype(np.float32): L.GG_W_F32,
                np.dtype(np.float64): L.GG_W_F64}[self.weights.dtype]

    def in_degree(self, v: int) -> int:
        return int(self.in_offsets[v + 1] - self.in_offsets[v])


class DeviceGraph:
    """A graph resident in HBM (gg_dev_graph). Create once, run many times."""

    def __init__(self, handle, n, e):
        self._h = C.c_void_p(handle) if not isinstance(handle, C.c_void_p) else handle
        self.n = int(n)
        self.e = int(e)

    @classmethod
    def upload(cls, g: Graph, device: int = -1, rank: int = 0, nranks: int = 1, exchange=None,
               for_run: "EngineConfig | None" = None):
        """for_run: the config of the one sparse-scheme run the graph is
        uploaded for -- its initial sparsification then overlaps the upload
        (gg_dev_graph_create_for_run)."""
        view = L.CscView(g.n, g.num_edges(), g.in_offsets.ctypes.data,
                         g.in_sources.ctypes.data if g.num_edges() else None,
                         g.weight_kind(),
                         g.weights.ctypes.data if g.weights is not None else None,
                         g.out_degree.ctypes.data if g.n else None)
        opts = L.PartOpts(device, rank, nranks, exchange)
        h = C.c_void_p()
        err = L.ErrorC()
        sch = None
        if for_run is not None:
            sch = (scheme_from_name(for_run.scheme) if isinstance(for_run.scheme, str)
                   else Scheme(for_run.scheme))
        if sch is not None and sch != Scheme.accurate and int(for_run.seed) >= 0:
            rc = L.lib().gg_dev_graph_create_for_run(C.byref(view), C.byref(opts),
                                                     float(for_run.sigma), int(for_run.seed),
                                                     C.byref(h), C.byref(err))
        else:
            rc = L.lib().gg_dev_graph_create(C.byref(view), C.byref(opts), C.byref(h), C.byref(err))
        _raise(rc, err)
        return cls(h, g.n, g.num_edges())

    @classmethod
    def load(cls, path, device: int = -1, rank: int = 0, nranks: int = 1, exchange=None):
        """Binary CSC file (reference GGCSR1 or GGCSR2) streamed straight to HBM."""
        opts = L.PartOpts(device, rank, nranks, exchange)
        h = C.c_void_p()
        err = L.ErrorC()
        rc = L.lib().gg_dev_graph_load(os.fsencode(path), C.byref(opts), C.byref(h), C.byref(err))
        if rc == L.GG_INVALID_ARGUMENT:
            raise RuntimeError(err.msg.decode())  # read_binary throws std::runtime_error
        _raise(rc, err)
        n, e = C.c_uint64(), C.c_uint64()
        L.lib().gg_dev_graph_info(h, C.byref(n), C.byref(e), None, None, None)
        dg = cls(h, n.value, e.value)
        dg.weight_dtype = {L.GG_W_U32: np.uint32, L.GG_W_F32: np.float32,
                           L.GG_W_F64: np.float64}.get(L.lib().gg_dev_graph_weight_kind(h))
        return dg

    def save(self, path):
        """GGCSR2 file (u32 sources, weight kind, out-degrees)."""
        err = L.ErrorC()
        _raise(L.lib().gg_dev_graph_save(self._h, os.fsencode(path), C.byref(err)), err)

    def last_projection(self) -> "DeviceView":
        """double[n] device projection of the last run (PR rank, SSSP distance,
        WCC label, BP belief[0]); valid until the next run on this graph."""
        p = C.c_void_p()
        _raise(L.lib().gg_last_projection(self._h, C.byref(p)), None)
        return DeviceView(p, self.n)

    @classmethod
    def rmat(cls, scale, edge_factor, seed, a=0.57, b=0.19, c=0.19, symmetrize=False,
             weights=None, device=-1, rank=0, nranks=1, exchange=None):
        """R-MAT generated straight into HBM (weights: None | 'u32' | 'coupling')."""
        wk = {None: L.GG_W_NONE, "u32": L.GG_W_U32, "coupling": L.GG_W_F32}[weights]
        p = L.RmatParams(scale, edge_factor, seed, a, b, c, int(symmetrize), wk)
        opts = L.PartOpts(device, rank, nranks, exchange)
        h = C.c_void_p()
        err = L.ErrorC()
        _raise(L.lib().gg_dev_graph_create_rmat(C.byref(p), C.byref(opts), C.byref(h),
                                                C.byref(err)), err)
        n, e = C.c_uint64(), C.c_uint64()
        L.lib().gg_dev_graph_info(h, C.byref(n), C.byref(e), None, None, None)
        out = cls(h, n.value, e.value)
        out.weight_dtype = {None: None, "u32": np.uint32, "coupling": np.float32}[weights]
        return out

    def symmetrized(self) -> "DeviceGraph":
        """graph.cpp:249-257 symmetrized(), built on the device (one rank)."""
        h = C.c_void_p()
        err = L.ErrorC()
        _raise(L.lib().gg_dev_graph_symmetrized(self._h, None, C.byref(h), C.byref(err)), err)
        out = DeviceGraph(h, self.n, 2 * self.e)
        out.weight_dtype = getattr(self, "weight_dtype", None)
        return out

    def info(self):
        vals = [C.c_uint64() for _ in range(5)]
        L.lib().gg_dev_graph_info(self._h, *[C.byref(v) for v in vals])
        return dict(zip(("n", "e", "v_begin", "v_end", "e_local"), (v.value for v in vals)))

    def to_host(self, alloc=None) -> Graph:
        """Copy the CSC back to host arrays made by alloc(count, dtype)
        (default np.empty; pass a pinned allocator for fast re-uploads)."""
        alloc = alloc or (lambda count, dt: np.empty(count, dt))
        n, e = self.n, self.e
        off = alloc(n + 1, np.uint64)
        src = alloc(max(e, 1), np.uint32)
        od = alloc(max(n, 1), np.uint32)
        wd = getattr(self, "weight_dtype", None)
        w = alloc(max(e, 1), wd) if wd is not None else None
        _raise(L.lib().gg_dev_graph_export(self._h, off.ctypes.data, src.ctypes.data,
                                           w.ctypes.data if w is not None else None,
                                           od.ctypes.data), None)
        return Graph(n, off, src[:e], None if w is None else w[:e], od[:n])

    def out_degree(self) -> np.ndarray:
        od = np.zeros(max(self.n, 1), np.uint32)
        _raise(L.lib().gg_dev_graph_export(self._h, None, None, None, od.ctypes.data), None)
        return od[:self.n]

    def close(self):
        if self._h:
            L.lib().gg_dev_graph_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# --------------------------------------------------------------------------
# Programs (algorithms.hpp) and factories (algorithms.cpp:71-98)
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class PageRankProgram:
    damping: float = 0.85
    epsilon: float = 1e-7


@dataclass(frozen=True)
class SsspProgram:
    source: int = 0
    graded: bool = False


@dataclass(frozen=True)
class WccProgram:
    pass


@dataclass(frozen=True)
class BeliefPropagationProgram:
    states: int = 2
    coupling: float = 0.8
    epsilon: float = 1e-6


@dataclass(frozen=True)
class EdgeBeliefPropagationProgram:
    """BASELINE C4: coupling per edge (the graph's weights), fp32 prior table
    (float32[n, 2] on the host, copied every run, or a DeviceBuffer kept
    resident), fp32 belief storage."""
    priors: object = field(default=None, repr=False, compare=False)
    epsilon: float = 1e-6


def pagerank_spec(damping: float = 0.85, epsilon: float = 1e-7) -> PageRankProgram:
    if not (0.0 < damping < 1.0):
        raise ValueError("pagerank damping must be in (0,1)")
    if not (epsilon > 0.0):
        raise ValueError("pagerank epsilon must be > 0")
    return PageRankProgram(damping, epsilon)


def sssp_spec(source: int, graded: bool = False) -> SsspProgram:
    return SsspProgram(source, graded)


def wcc_spec() -> WccProgram:
    return WccProgram()


def bp_spec(states: int = 2, coupling: float = 0.8, epsilon: float = 1e-6):
    if states < 2:
        raise ValueError("bp states must be >= 2")
    if not (0.0 < coupling < 1.0):
        raise ValueError("bp coupling must be in (0,1)")
    if not (epsilon > 0.0):
        raise ValueError("bp epsilon must be > 0")
    return BeliefPropagationProgram(states, coupling, epsilon)


# --------------------------------------------------------------------------
# Engine
# --------------------------------------------------------------------------
@dataclass
class EngineConfig:
    scheme: Scheme | str = Scheme.accurate
    sigma: float = 1.0
    theta: float = 0.0
    alpha: int = 1
    max_iterations: int = 100
    seed: int = 0
    threads: int = 1

    def c(self) -> L.EngineConfigC:
        s = scheme_from_name(self.scheme) if isinstance(self.scheme, str) else Scheme(self.scheme)
        if self.alpha < 0 or self.max_iterations < 0 or self.threads < 0:
            raise ValueError("alpha, max_iterations and threads must be non-negative")
        return L.EngineConfigC(int(s), float(self.sigma), float(self.theta), int(self.alpha),
                               int(self.max_iterations), int(self.seed), int(self.threads))


@dataclass
class IterationRecord:
    mode: IterationMode
    processed_edges: int
    active_vertices: int
    wall_seconds: float
    kernel_ms: float = 0.0
    rebuild_ms: float = 0.0
    exchange_ms: float = 0.0
    algo_bytes: int = 0
    edge_ms: float = 0.0
    vertex_ms: float = 0.0
    edge_bytes: int = 0
    vertex_bytes: int = 0


@dataclass
class RunReport:
    final_properties: np.ndarray
    iterations_run: int
    per_iteration: list
    total_wall_seconds: float
    total_processed_edges: int
    kept_edges: int = 0
    kernel_launches: int = 0
    flags: np.ndarray | None = None  # final active-edge flags, one byte per edge (when requested)
    flag_words: np.ndarray | None = None  # the same flags as the device bitmap (uint32 words)
    exchange_fused: bool = False  # several ranks: messages stored into the peer replicas


def validate(cfg: EngineConfig) -> None:
    err = L.ErrorC()
    _raise(L.lib().gg_validate(C.byref(cfg.c()), C.byref(err)), err)


def mode_for(scheme, t: int, alpha: int) -> IterationMode:
    s = scheme_from_name(scheme) if isinstance(scheme, str) else int(scheme)
    return IterationMode(L.lib().gg_mode_for(int(s), t, alpha))


def select_superstep_iterations(alpha: int, max_iterations: int, scheme) -> list:
    if alpha < 1:
        raise ValueError("alpha must be >= 1")
    s = scheme_from_name(scheme) if isinstance(scheme, str) else int(scheme)
    k = L.lib().gg_select_superstep_iterations(alpha, max_iterations, int(s), None, 0)
    out = np.zeros(max(k, 1), np.uint64)
    L.lib().gg_select_superstep_iterations(alpha, max_iterations, int(s), out.ctypes.data, k)
    return [int(x) for x in out[:k]]


def sparsify(graph_or_e, sigma: float, seed: int) -> np.ndarray:
    """engine.cpp:63-75 on the device; returns one flag byte per edge."""
    e = graph_or_e.num_edges() if isinstance(graph_or_e, Graph) else int(graph_or_e)
    words = np.zeros(max((e + 31) // 32, 1), np.uint32)
    err = L.ErrorC()
    _raise(L.lib().gg_sparsify(e, float(sigma), int(seed), words.ctypes.data, C.byref(err)), err)
    return unpack_bitmap(words, e)


def unpack_bitmap(words: np.ndarray, e: int) -> np.ndarray:
    return np.unpackbits(words.view(np.uint8), bitorder="little")[:e].astype(np.uint8)


def _out_buffer(out, shape, dtype):
    if out is None:
        return np.zeros(shape, dtype)
    if out.dtype != np.dtype(dtype) or out.shape != (shape if isinstance(shape, tuple) else (shape,)) \
            or not out.flags["C_CONTIGUOUS"]:
        raise ValueError(f"out must be a C-contiguous {np.dtype(dtype).name} array of shape {shape}")
    return out


def run(graph, program, cfg: EngineConfig, *, want_flags: bool = False, timing: bool = False,
        rec_cap: int | None = None, device_output: bool = False, out=None,
        grid_ctas: int = 0) -> RunReport:
    """gg::run (engine.hpp:141-249) on the device. `graph` is a Graph
    (uploaded for the call) or a DeviceGraph (already resident).
    timing: CUDA-event time of every kernel into the records.
    device_output: leave the final properties in HBM (no D2H copy;
    final_properties is then None).
    out: caller-owned result array (e.g. pinned host memory) of the
    program's property shape/dtype, filled instead of a fresh array.
    grid_ctas: test hook, caps the CTAs of every engine launch (0 = the
    occupancy-sized grid); results are identical for any value."""
    ccfg = cfg.c()
    owned = None
    if isinstance(graph, Graph):  # gg::run(Graph, ...): upload for this run
        dg = owned = DeviceGraph.upload(graph, for_run=cfg)
        n, e = graph.n, graph.num_edges()
    else:
        dg = graph
        n, e = graph.n, graph.e
    try:
        cap = rec_cap if rec_cap is not None else int(min(max(cfg.max_iterations, 1), 1 << 16))
        recs = (L.IterRecordC * max(cap, 1))()
        summ = L.RunSummaryC()
        flags = np.zeros(max((e + 31) // 32, 1), np.uint32) if want_flags else None
        opts = L.RunOptsC(flags.ctypes.data if flags is not None else None, int(timing),
                          int(device_output), int(grid_ctas))
        err = L.ErrorC()
        lib = L.lib()
        if isinstance(program, PageRankProgram):
            props = _out_buffer(out, n, np.float64)
            p = L.PrParams(program.damping, program.epsilon)
            rc = lib.gg_run_pr(dg._h, C.byref(ccfg), C.byref(p), props.ctypes.data, recs, cap,
                               C.byref(summ), C.byref(opts), C.byref(err))
        elif isinstance(program, SsspProgram):
            props = _out_buffer(out, n, np.float64)
            p = L.SsspParams(program.source, int(program.graded))
            rc = lib.gg_run_sssp(dg._h, C.byref(ccfg), C.byref(p), props.ctypes.data, recs, cap,
                                 C.byref(summ), C.byref(opts), C.byref(err))
        elif isinstance(program, WccProgram):
            props = _out_buffer(out, n, np.uint32)
            rc = lib.gg_run_wcc(dg._h, C.byref(ccfg), props.ctypes.data, recs, cap,
                                C.byref(summ), C.byref(opts), C.byref(err))
        elif isinstance(program, BeliefPropagationProgram):
            props = _out_buffer(out, (n, program.states), np.float64)
            p = L.BpParams(program.states, program.coupling, program.epsilon, None, 0)
            rc = lib.gg_run_bp(dg._h, C.byref(ccfg), C.byref(p), props.ctypes.data, recs, cap,
                               C.byref(summ), C.byref(opts), C.byref(err))
        elif isinstance(program, EdgeBeliefPropagationProgram):
            props = _out_buffer(out, (n, 2), np.float64)
            if isinstance(program.priors, DeviceBuffer):
                if program.priors.nbytes < 8 * n:
                    raise ValueError("edge BP needs a float32[n, 2] prior table")
                p = L.BpParams(2, 0.0, program.epsilon, program.priors.ptr, 1)
            else:
                pri = np.ascontiguousarray(program.priors, np.float32).reshape(-1)
                if pri.shape[0] != 2 * n:
                    raise ValueError("edge BP needs a float32[n, 2] prior table")
                p = L.BpParams(2, 0.0, program.epsilon, pri.ctypes.data, 0)
            rc = lib.gg_run_bp(dg._h, C.byref(ccfg), C.byref(p), props.ctypes.data, recs, cap,
                               C.byref(summ), C.byref(opts), C.byref(err))
        else:
            raise TypeError(f"no device program for {type(program).__name__} "
                            "(programs: PageRank, SSSP, WCC, BP, edge-BP)")
        _raise(rc, err)
        k = int(min(summ.iterations_run, cap))
        per = [IterationRecord(IterationMode(recs[i].mode), int(recs[i].processed_edges),
                               int(recs[i].active_vertices), float(recs[i].wall_seconds),
                               float(recs[i].kernel_ms), float(recs[i].rebuild_ms),
                               float(recs[i].exchange_ms), int(recs[i].algo_bytes),
                               float(recs[i].edge_ms), float(recs[i].vertex_ms),
                               int(recs[i].edge_bytes), int(recs[i].vertex_bytes))
               for i in range(k)]
        out_props = None if device_output else (props if n else props[:0])
        return RunReport(out_props, int(summ.iterations_run), per,
                         float(summ.total_wall_seconds), int(summ.total_processed_edges),
                         int(summ.kept_edges), int(summ.kernel_launches),
                         unpack_bitmap(flags, e) if flags is not None else None, flags,
                         bool(summ.exchange_fused))
    finally:
        if owned is not None:
            owned.close()


# --------------------------------------------------------------------------
# Metrics (metrics.hpp / metrics.cpp) — host C++ in libggb.so
# --------------------------------------------------------------------------
@dataclass
class ErrorReport:
    metric: str
    error: float
    accuracy: float
    k: int = 0


def _on_device(*xs):
    dev = [isinstance(x, (DeviceView, DeviceBuffer)) for x in xs]
    if any(dev) and not all(dev):
        raise TypeError("metric inputs must both be host arrays or both device arrays")
    if all(dev) and xs[0].n != xs[1].n:
        raise ValueError("metric inputs have different lengths")
    return all(dev)


def _metric_args(approx, exact):
    a = np.ascontiguousarray(approx, np.float64)
    x = np.ascontiguousarray(exact, np.float64)
    if a.shape != x.shape:
        raise ValueError("metric inputs have different lengths")
    return a, x


def topk_error(approx, exact, k: int) -> ErrorReport:
    """metrics.cpp:60-72; host arrays, or device arrays (DeviceView /
    DeviceBuffer: computed on the GPU, only the scalar comes back)."""
    out = C.c_double()
    if _on_device(approx, exact):
        _raise(L.lib().gg_topk_error_dev(approx.ptr, exact.ptr, approx.n, int(k), C.byref(out)), None)
        return ErrorReport("topk", out.value, (1.0 - out.value) * 100.0, int(k))
    a, x = _metric_args(approx, exact)
    _raise(L.lib().gg_topk_error(a.ctypes.data, x.ctypes.data, len(a), int(k), C.byref(out)), None)
    return ErrorReport("topk", out.value, (1.0 - out.value) * 100.0, int(k))


def relative_error(approx, exact) -> ErrorReport:
    out = C.c_double()
    if _on_device(approx, exact):
        _raise(L.lib().gg_relative_error_dev(approx.ptr, exact.ptr, approx.n, C.byref(out)), None)
        return ErrorReport("relative", out.value, (1.0 - out.value) * 100.0)
    a, x = _metric_args(approx, exact)
    _raise(L.lib().gg_relative_error(a.ctypes.data, x.ctypes.data, len(a), C.byref(out)), None)
    return ErrorReport("relative", out.value, (1.0 - out.value) * 100.0)


def stretch_error(approx, exact) -> ErrorReport:
    out = C.c_double()
    if _on_device(approx, exact):
        err = L.ErrorC()
        rc = L.lib().gg_stretch_error_dev(approx.ptr, exact.ptr, approx.n, C.byref(out), C.byref(err))
        if rc == L.GG_INVALID_ARGUMENT:
            raise RuntimeError(err.msg.decode())
        _raise(rc, err)
        return ErrorReport("stretch", out.value, (1.0 - out.value) * 100.0)
    a, x = _metric_args(approx, exact)
    rc = L.lib().gg_stretch_error(a.ctypes.data, x.ctypes.data, len(a), C.byref(out))
    if rc == L.GG_INVALID_ARGUMENT:
        raise RuntimeError("stretch_error: approximate distance below exact (engine bug)")
    _raise(rc, None)
    return ErrorReport("stretch", out.value, (1.0 - out.value) * 100.0)


class Exchange:
    """NCCL transport of the 1-D destination partition (one process per GPU).
    Rank 0 makes the id (Exchange.unique_id()); the caller broadcasts it
    (e.g. torch.distributed.broadcast_object_list) and every rank builds
    Exchange(rank, nranks, uid) before creating its DeviceGraph."""

    def __init__(self, rank: int, nranks: int, uid: bytes):
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        err = L.ErrorC()
        _raise(L.lib().gg_exchange_nccl_create(buf, rank, nranks, C.byref(h), C.byref(err)), err)
        self.handle = h
        self.rank, self.nranks = rank, nranks

    @classmethod
    def local_group(cls, nranks: int) -> list["Exchange"]:
        """In-process transport: one handle per rank for ranks run as threads of
        this process (each with its own DeviceGraph; one GPU may host all)."""
        hs = (C.c_void_p * nranks)()
        _raise(L.lib().gg_exchange_local_group(nranks, hs), None)
        out = []
        for r in range(nranks):
            x = cls.__new__(cls)
            x.handle = C.c_void_p(hs[r])
            x.rank, x.nranks = r, nranks
            out.append(x)
        return out

    def set_fused(self, on: bool) -> None:
        """Fused exchange (default on): the vertex kernel stores the new
        messages into every rank's replica over peer memory; off: all-gather
        after it. Same value on every rank (gg_exchange_set_fused)."""
        _raise(L.lib().gg_exchange_set_fused(self.handle, 1 if on else 0), None)

    def selftest(self) -> None:
        """Collective transport check (gg_exchange_selftest): ragged all-gather
        and all-reduces over the communicator against their closed forms;
        raises on any difference. Every rank calls it."""
        err = L.ErrorC()
        _raise(L.lib().gg_exchange_selftest(self.handle, C.byref(err)), err)

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        _raise(L.lib().gg_nccl_unique_id(buf), None)
        return bytes(buf)

    def close(self):
        if self.handle:
            L.lib().gg_exchange_destroy(self.handle)
            self.handle = C.c_void_p()


class DeviceView:
    """Non-owning double[n] device array, e.g. DeviceGraph.last_projection()
    (valid until the graph's next run; DeviceBuffer.copy keeps it)."""

    def __init__(self, ptr, n: int):
        self.ptr = ptr
        self.n = int(n)
        self.nbytes = 8 * self.n


class DeviceBuffer:
    """Device memory owned by libggb (gg_device_upload / gg_bp_priors_device)."""

    def __init__(self, ptr, nbytes: int):
        self.ptr = ptr
        self.nbytes = int(nbytes)
        self.n = self.nbytes // 8

    @classmethod
    def copy(cls, view) -> "DeviceBuffer":
        h = C.c_void_p()
        _raise(L.lib().gg_device_copy(view.ptr, view.nbytes, C.byref(h)), None)
        return cls(h, view.nbytes)

    @classmethod
    def upload(cls, array: np.ndarray) -> "DeviceBuffer":
        a = np.ascontiguousarray(array)
        h = C.c_void_p()
        _raise(L.lib().gg_device_upload(a.ctypes.data, a.nbytes, C.byref(h)), None)
        return cls(h, a.nbytes)

    def close(self):
        if self.ptr:
            L.lib().gg_device_free(self.ptr)
            self.ptr = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def bp_priors(n: int, seed: int, device: bool = False):
    """BASELINE C4 priors generated on the device: float32[n, 2] on the host,
    or (device=True) a DeviceBuffer that stays resident."""
    if device:
        h = C.c_void_p()
        _raise(L.lib().gg_bp_priors_device(n, seed, C.byref(h)), None)
        return DeviceBuffer(h, 8 * n)
    out = np.zeros(2 * max(n, 1), np.float32)
    _raise(L.lib().gg_bp_priors(n, seed, out.ctypes.data), None)
    return out[:2 * n].reshape(n, 2)


def partition_plan(g: Graph, nranks: int) -> np.ndarray:
    out = np.zeros(nranks + 1, np.uint64)
    _raise(L.lib().gg_partition_plan(g.n, g.in_offsets.ctypes.data, nranks, out.ctypes.data), None)
    return out
