"""ctypes face of the CPU CHECKERS — TEST INFRASTRUCTURE ONLY.

* ``Oracle``     wraps oracle/liboracle.so (plain-C restatement, gg_oracle.c).
* ``Reference``  wraps oracle/_ref/libggref.so (the unmodified reference
  compiled from /root/reference by oracle/Makefile; may be absent on a box
  that never had /root/reference — then ``Reference.available()`` is False).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libggref.so")

ACCURATE, SP, SMS, GG = 0, 1, 2, 3
SCHEMES = {"accurate": ACCURATE, "sp": SP, "sms": SMS, "gg": GG}
MODE_NAMES = ("approximate", "accurate", "superstep")
PR, SSSP, WCC, BP, BP_EDGE, POISON = 0, 1, 2, 3, 4, 5

u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")


class _Graph(C.Structure):
    _fields_ = [("n", C.c_uint64), ("e", C.c_uint64), ("off", C.POINTER(C.c_uint64)),
                ("src", C.POINTER(C.c_uint32)), ("w", C.POINTER(C.c_double)),
                ("outdeg", C.POINTER(C.c_uint32))]


class _Config(C.Structure):
    _fields_ = [("scheme", C.c_int), ("sigma", C.c_double), ("theta", C.c_double),
                ("alpha", C.c_uint64), ("max_iterations", C.c_uint64), ("seed", C.c_uint64),
                ("threads", C.c_uint32)]


class _Params(C.Structure):
    _fields_ = [("damping", C.c_double), ("epsilon", C.c_double), ("source", C.c_uint32),
                ("graded", C.c_int), ("states", C.c_int), ("coupling", C.c_double),
                ("prior_table", C.c_void_p), ("poison_vertex", C.c_uint32),
                ("poison_iteration", C.c_int)]


class _Record(C.Structure):
    _fields_ = [("mode", C.c_int32), ("processed_edges", C.c_uint64),
                ("active_vertices", C.c_uint64)]


class _Summary(C.Structure):
    _fields_ = [("iterations_run", C.c_uint64), ("total_processed_edges", C.c_uint64),
                ("err_iteration", C.c_uint64), ("err_vertex", C.c_uint32)]


class _Lockstep(C.Structure):
    _fields_ = [("dev_bitmaps", C.POINTER(C.c_void_p)), ("n_dev", C.c_uint64),
                ("tol_unit", C.c_double), ("stats", C.POINTER(C.c_uint64)),
                ("stats_cap", C.c_uint64), ("n_supersteps", C.c_uint64)]


class _RefRecord(C.Structure):
    _fields_ = [("mode", C.c_int32), ("processed_edges", C.c_uint64),
                ("active_vertices", C.c_uint64), ("wall_seconds", C.c_double)]


class _RefSummary(C.Structure):
    _fields_ = [("iterations_run", C.c_uint64), ("total_processed_edges", C.c_uint64),
                ("err_iteration", C.c_uint64), ("err_vertex", C.c_uint32),
                ("total_wall_seconds", C.c_double)]


@dataclass
class CSC:
    """Host pull CSC (gg::Graph layout, graph.hpp:29-49)."""
    n: int
    off: np.ndarray            # uint64[n+1]
    src: np.ndarray            # uint32[e]
    w: np.ndarray | None = None  # float64[e] or None
    outdeg: np.ndarray | None = None

    def __post_init__(self):
        self.off = np.ascontiguousarray(self.off, dtype=np.uint64)
        self.src = np.ascontiguousarray(self.src, dtype=np.uint32)
        if self.w is not None:
            self.w = np.ascontiguousarray(self.w, dtype=np.float64)
        if self.outdeg is None:
            self.outdeg = np.bincount(self.src, minlength=self.n).astype(np.uint32) \
                if self.n else np.zeros(0, np.uint32)
        self.outdeg = np.ascontiguousarray(self.outdeg, dtype=np.uint32)

    @property
    def e(self) -> int:
        return int(self.src.shape[0])


@dataclass
class Result:
    status: int
    props: np.ndarray | None
    modes: list = field(default_factory=list)
    processed_edges: list = field(default_factory=list)
    active_vertices: list = field(default_factory=list)
    wall_seconds: list = field(default_factory=list)
    iterations_run: int = 0
    total_processed_edges: int = 0
    err_iteration: int = 0
    err_vertex: int = 0
    msg: str = ""
    flags: np.ndarray | None = None
    # lock-step runs: per superstep {near, adopted, real, kept} (gg_oracle.h og_lockstep)
    lockstep: list = field(default_factory=list)


def _params(prog, damping=0.85, epsilon=None, source=0, graded=False, states=2,
            coupling=0.8, prior_table=None, poison_vertex=2, poison_iteration=3):
    if epsilon is None:
        epsilon = 1e-6 if prog in (BP, BP_EDGE) else 1e-7
    p = _Params(damping, epsilon, source, int(graded), states, coupling, None,
                poison_vertex, poison_iteration)
    if prior_table is not None:
        p.prior_table = prior_table.ctypes.data
    return p


def _prop_shape(prog, n, states):
    if prog == WCC:
        return np.zeros(n, np.uint32)
    if prog == BP:
        return np.zeros((n, states), np.float64)
    if prog == BP_EDGE:
        return np.zeros((n, 2), np.float64)
    return np.zeros(n, np.float64)


class Oracle:
    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not os.path.exists(ORACLE_SO):
                raise RuntimeError(f"oracle not built: {ORACLE_SO} (run __graft_entry__.build())")
            L = C.CDLL(ORACLE_SO)
            G = C.POINTER(_Graph)
            for name, argt in {
                "og_build_graph": [C.c_uint64, C.c_uint64, u32p, u32p, C.c_void_p],
                "og_from_csc": [C.c_uint64, C.c_uint64, u64p, u32p, C.c_void_p],
                "og_generate_dumbbell": [C.c_uint64],
                "og_generate_power_law": [C.c_uint64, C.c_double, C.c_double, C.c_uint64],
                "og_random_graph": [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int],
                "og_symmetrized": [G], "og_reverse": [G],
                "og_rmat": [C.c_uint32, C.c_uint32, C.c_uint64, C.c_double, C.c_double,
                            C.c_double, C.c_int],
            }.items():
                getattr(L, name).argtypes = argt
                getattr(L, name).restype = G
            L.og_free_graph.argtypes = [G]
            L.og_rmat_weights_u32.argtypes = [C.c_uint64, C.c_uint64, u32p]
            L.og_bp_priors.argtypes = [C.c_uint64, C.c_uint64, f32p]
            L.og_bp_couplings.argtypes = [C.c_uint64, C.c_uint64, f32p]
            L.og_max_outdeg_vertex.argtypes = [G]
            L.og_max_outdeg_vertex.restype = C.c_uint32
            L.og_sparsify.argtypes = [C.c_uint64, C.c_double, C.c_uint64, u8p]
            L.og_mode_for.argtypes = [C.c_int, C.c_uint64, C.c_uint64]
            L.og_supersteps.argtypes = [C.c_uint64, C.c_uint64, C.c_int, u64p, C.c_uint64]
            L.og_supersteps.restype = C.c_uint64
            L.og_run.argtypes = [G, C.c_int, C.POINTER(_Params), C.POINTER(_Config), C.c_void_p,
                                 C.POINTER(_Record), C.c_uint64, C.POINTER(_Summary), C.c_void_p,
                                 C.c_char_p, C.c_size_t]
            L.og_run_ex.argtypes = L.og_run.argtypes + [C.POINTER(_Lockstep)]
            L.og_influences.argtypes = [G, C.c_int, C.POINTER(_Params), C.c_void_p, C.c_uint64,
                                        C.c_uint64, C.c_int, f64p]
            L.og_mix64.argtypes = [C.c_uint64]
            L.og_mix64.restype = C.c_uint64
            L.og_init_props.argtypes = [G, C.c_int, C.POINTER(_Params), C.c_void_p]
            L.og_step_range.argtypes = [G, C.c_int, C.POINTER(_Params), C.c_int, C.c_double,
                                        u8p, u32p, C.c_void_p, u8p, C.c_void_p, u8p, C.c_uint64,
                                        C.c_uint64, u64p]
            for m in ("og_relative_error", "og_stretch_error"):
                getattr(L, m).argtypes = [f64p, f64p, C.c_uint64, C.POINTER(C.c_double)]
            L.og_topk_error.argtypes = [f64p, f64p, C.c_uint64, C.c_uint64, C.POINTER(C.c_double)]
            cls._lib = L
        return cls._lib

    # -- graphs -------------------------------------------------------------
    @classmethod
    def _take(cls, gp) -> CSC:
        if not gp:
            raise ValueError("oracle graph construction failed")
        g = gp.contents
        n, e = int(g.n), int(g.e)
        off = np.ctypeslib.as_array(g.off, shape=(n + 1,)).copy()
        src = np.ctypeslib.as_array(g.src, shape=(e,)).copy() if e else np.zeros(0, np.uint32)
        w = np.ctypeslib.as_array(g.w, shape=(e,)).copy() if (g.w and e) else None
        od = np.ctypeslib.as_array(g.outdeg, shape=(n,)).copy() if n else np.zeros(0, np.uint32)
        cls.lib().og_free_graph(gp)
        return CSC(n, off, src, w, od)

    @classmethod
    def _view(cls, g: CSC):
        """An og_graph over the CSC's own arrays (no copy; the CSC must
        outlive the returned struct)."""
        v = _Graph(g.n, g.e, g.off.ctypes.data_as(C.POINTER(C.c_uint64)),
                   g.src.ctypes.data_as(C.POINTER(C.c_uint32)),
                   g.w.ctypes.data_as(C.POINTER(C.c_double)) if g.w is not None else None,
                   g.outdeg.ctypes.data_as(C.POINTER(C.c_uint32)))
        return v

    @classmethod
    def _ptr(cls, g: CSC):
        return cls.lib().og_from_csc(g.n, g.e, g.off, g.src,
                                     g.w.ctypes.data if g.w is not None else None)

    @classmethod
    def build_graph(cls, n, src, dst, w=None) -> CSC:
        src = np.ascontiguousarray(src, np.uint32)
        dst = np.ascontiguousarray(dst, np.uint32)
        wp = None
        if w is not None:
            w = np.ascontiguousarray(w, np.float64)
            wp = w.ctypes.data
        return cls._take(cls.lib().og_build_graph(n, len(src), src, dst, wp))

    @classmethod
    def dumbbell(cls, k) -> CSC:
        return cls._take(cls.lib().og_generate_dumbbell(k))

    @classmethod
    def power_law(cls, n, avg, ex, seed) -> CSC:
        return cls._take(cls.lib().og_generate_power_law(n, avg, ex, seed))

    @classmethod
    def random_graph(cls, n, m, seed, weighted=False) -> CSC:
        return cls._take(cls.lib().og_random_graph(n, m, seed, int(weighted)))

    @classmethod
    def symmetrized(cls, g: CSC) -> CSC:
        p = cls._ptr(g)
        r = cls._take(cls.lib().og_symmetrized(p))
        cls.lib().og_free_graph(p)
        return r

    @classmethod
    def reverse(cls, g: CSC) -> CSC:
        p = cls._ptr(g)
        r = cls._take(cls.lib().og_reverse(p))
        cls.lib().og_free_graph(p)
        return r

    @classmethod
    def rmat(cls, scale, edge_factor, seed, a=0.57, b=0.19, c=0.19, threads=0) -> CSC:
        return cls._take(cls.lib().og_rmat(scale, edge_factor, seed, a, b, c, threads))

    @classmethod
    def rmat_weights_u32(cls, e, seed):
        out = np.zeros(e, np.uint32)
        cls.lib().og_rmat_weights_u32(e, seed, out)
        return out

    @classmethod
    def bp_priors(cls, n, seed):
        out = np.zeros(2 * n, np.float32)
        cls.lib().og_bp_priors(n, seed, out)
        return out

    @classmethod
    def bp_couplings(cls, e, seed):
        out = np.zeros(e, np.float32)
        cls.lib().og_bp_couplings(e, seed, out)
        return out

    @classmethod
    def max_outdeg_vertex(cls, g: CSC) -> int:
        return int(np.argmax(g.outdeg)) if g.n else 0

    # -- engine -------------------------------------------------------------
    @classmethod
    def sparsify(cls, e, sigma, seed):
        out = np.zeros(max(e, 1), np.uint8)
        rc = cls.lib().og_sparsify(e, sigma, seed, out)
        if rc:
            raise ValueError("sigma must be in [0,1]")
        return out[:e]

    @classmethod
    def mode_for(cls, scheme, t, alpha):
        return cls.lib().og_mode_for(scheme, t, alpha)

    @classmethod
    def supersteps(cls, alpha, max_it, scheme):
        out = np.zeros(4096, np.uint64)
        k = cls.lib().og_supersteps(alpha, max_it, scheme, out, len(out))
        return [int(x) for x in out[:min(k, len(out))]]

    @classmethod
    def run(cls, g: CSC, prog, scheme=ACCURATE, sigma=1.0, theta=0.0, alpha=1,
            max_iterations=100, seed=0, threads=1, want_flags=False, device_flags=None,
            tol_unit=None, **pp) -> Result:
        """og_run. Lock-step (og_run_ex) when `tol_unit` is given:
        `device_flags` = the device's flag bitmaps (uint32 words) right
        after each superstep, in order (None entries: no comparison); edges
        within the near-threshold band whose device flag differs are
        adopted, others are counted as real mismatches (Result.lockstep)."""
        L = cls.lib()
        params = _params(prog, **pp)
        cfg = _Config(scheme, sigma, theta, alpha, max_iterations, seed, threads)
        cap = max_iterations if max_iterations < (1 << 20) else (1 << 20)
        cap = max(1, min(cap, 1 << 20))
        recs = (_Record * cap)()
        summ = _Summary()
        props = _prop_shape(prog, g.n, pp.get("states", 2))
        flags = np.zeros(max(g.e, 1), np.uint8) if want_flags else None
        msg = C.create_string_buffer(256)
        gv = cls._view(g)
        args = [C.byref(gv), prog, C.byref(params), C.byref(cfg), props.ctypes.data, recs, cap,
                C.byref(summ), flags.ctypes.data if flags is not None else None, msg, 256]
        stats_out = []
        if tol_unit is None:
            rc = L.og_run(*args)
        else:
            dev = [None if d is None else np.ascontiguousarray(d, np.uint32) for d in
                   (device_flags or [])]
            ptrs = (C.c_void_p * max(len(dev), 1))(*[d.ctypes.data if d is not None else None
                                                       for d in dev])
            scap = max(len(dev), max_iterations if max_iterations < 4096 else 4096, 1)
            stats = np.zeros(4 * scap, np.uint64)
            ls = _Lockstep(ptrs, len(dev), float(tol_unit),
                           stats.ctypes.data_as(C.POINTER(C.c_uint64)), scap, 0)
            rc = L.og_run_ex(*args, C.byref(ls))
            for i in range(min(int(ls.n_supersteps), scap)):
                near, adopted, real, kept = (int(x) for x in stats[4 * i:4 * i + 4])
                stats_out.append(dict(near=near, adopted=adopted, real=real, kept=kept,
                                      compared=i < len(dev) and dev[i] is not None))
        k = int(min(summ.iterations_run, cap))
        return Result(rc, props, [int(recs[i].mode) for i in range(k)],
                      [int(recs[i].processed_edges) for i in range(k)],
                      [int(recs[i].active_vertices) for i in range(k)], [],
                      int(summ.iterations_run), int(summ.total_processed_edges),
                      int(summ.err_iteration), int(summ.err_vertex), msg.value.decode(),
                      flags[:g.e] if flags is not None else None, stats_out)

    @classmethod
    def influences(cls, g: CSC, prog, prev, v_begin=0, v_end=None, threads=1, **pp):
        """Per-edge superstep influences of destinations [v_begin, v_end)
        from properties `prev` (og_influences)."""
        v_end = g.n if v_end is None else v_end
        params = _params(prog, **pp)
        out = np.zeros(max(int(g.off[v_end] - g.off[v_begin]), 1), np.float64)
        prev = np.ascontiguousarray(prev)
        gv = cls._view(g)
        if cls.lib().og_influences(C.byref(gv), prog, C.byref(params), prev.ctypes.data, v_begin,
                                   v_end, threads, out):
            raise ValueError("og_influences failed")
        return out[:int(g.off[v_end] - g.off[v_begin])]

    # -- per-range step (multi-rank protocol tests) ----------------------------
    class Stepper:
        """Holds an oracle graph and runs og_step_range on numpy state."""

        def __init__(self, g: CSC, prog, **pp):
            self.g, self.prog = g, prog
            self.params = _params(prog, **pp)
            self.gp = Oracle._ptr(g)
            self.states = pp.get("states", 2)

        def init_props(self):
            props = _prop_shape(self.prog, self.g.n, self.states)
            Oracle.lib().og_init_props(self.gp, self.prog, C.byref(self.params), props.ctypes.data)
            return props

        def step(self, mode, theta, flags, aid, prev, status, nxt, status_next, vb, ve):
            ctr = np.zeros(4, np.uint64)
            rc = Oracle.lib().og_step_range(self.gp, self.prog, C.byref(self.params), mode, theta,
                                            flags, aid, prev.ctypes.data, status, nxt.ctypes.data,
                                            status_next, vb, ve, ctr)
            if rc:
                raise ValueError("og_step_range failed")
            return ctr

        def close(self):
            if self.gp:
                Oracle.lib().og_free_graph(self.gp)
                self.gp = None

    # -- metrics ------------------------------------------------------------
    @classmethod
    def topk_error(cls, approx, exact, k):
        r = C.c_double()
        a = np.ascontiguousarray(approx, np.float64); x = np.ascontiguousarray(exact, np.float64)
        if cls.lib().og_topk_error(a, x, len(a), k, C.byref(r)):
            raise ValueError("topk k must be in [1, N]")
        return r.value

    @classmethod
    def relative_error(cls, approx, exact):
        r = C.c_double()
        a = np.ascontiguousarray(approx, np.float64); x = np.ascontiguousarray(exact, np.float64)
        cls.lib().og_relative_error(a, x, len(a), C.byref(r))
        return r.value

    @classmethod
    def stretch_error(cls, approx, exact):
        r = C.c_double()
        a = np.ascontiguousarray(approx, np.float64); x = np.ascontiguousarray(exact, np.float64)
        if cls.lib().og_stretch_error(a, x, len(a), C.byref(r)):
            raise RuntimeError("stretch_error: approximate distance below exact")
        return r.value


class Reference:
    """The unmodified reference (oracle/_ref/libggref.so)."""
    _lib = None

    @classmethod
    def available(cls) -> bool:
        return os.path.exists(REF_SO)

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not cls.available():
                raise RuntimeError(f"reference build missing: {REF_SO}")
            L = C.CDLL(REF_SO)
            L.ref_graph_create.argtypes = [C.c_uint64, C.c_uint64, u64p, u32p, C.c_void_p]
            L.ref_graph_create.restype = C.c_void_p
            L.ref_graph_destroy.argtypes = [C.c_void_p]
            L.ref_run.argtypes = [C.c_void_p, C.c_int, C.POINTER(_Params), C.POINTER(_Config),
                                  C.c_void_p, C.POINTER(_RefRecord), C.c_uint64,
                                  C.POINTER(_RefSummary), C.c_void_p, C.c_char_p, C.c_size_t]
            L.ref_sparsify.argtypes = [C.c_void_p, C.c_double, C.c_uint64, u8p]
            L.ref_mode_for.argtypes = [C.c_int, C.c_uint64, C.c_uint64]
            L.ref_supersteps.argtypes = [C.c_uint64, C.c_uint64, C.c_int, u64p, C.c_uint64]
            L.ref_supersteps.restype = C.c_uint64
            for nm in ("ref_generate_dumbbell",):
                getattr(L, nm).argtypes = [C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
                getattr(L, nm).restype = C.c_void_p
            L.ref_generate_power_law.argtypes = [C.c_uint64, C.c_double, C.c_double, C.c_uint64,
                                                 C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
            L.ref_generate_power_law.restype = C.c_void_p
            L.ref_symmetrized.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
            L.ref_symmetrized.restype = C.c_void_p
            L.ref_graph_arrays.argtypes = [C.c_void_p, u64p, u32p, C.c_void_p, u32p]
            L.ref_graph_weighted.argtypes = [C.c_void_p]
            L.ref_write_binary.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p, C.c_size_t]
            L.ref_read_binary.argtypes = [C.c_char_p, C.POINTER(C.c_uint64),
                                          C.POINTER(C.c_uint64), C.c_char_p, C.c_size_t]
            L.ref_read_binary.restype = C.c_void_p
            L.ref_metric.argtypes = [C.c_int, f64p, f64p, C.c_uint64, C.c_uint64,
                                     C.POINTER(C.c_double)]
            L.ref_sweep_csv.argtypes = [C.c_void_p, C.c_char_p, C.c_int, C.c_int, f64p, C.c_int,
                                        f64p, C.c_int, u64p, C.c_int, C.c_uint64, C.c_int, u64p,
                                        C.c_int, C.c_uint32, C.c_int, C.c_double, C.c_char_p,
                                        C.c_size_t]
            L.ref_sweep_csv.restype = C.c_long
            cls._lib = L
        return cls._lib

    @classmethod
    def graph(cls, g: CSC):
        return cls.lib().ref_graph_create(g.n, g.e, g.off, g.src,
                                          g.w.ctypes.data if g.w is not None else None)

    @classmethod
    def free(cls, h):
        cls.lib().ref_graph_destroy(h)

    @classmethod
    def _export(cls, h, n, e) -> CSC:
        L = cls.lib()
        off = np.zeros(n + 1, np.uint64); src = np.zeros(max(e, 1), np.uint32)
        od = np.zeros(max(n, 1), np.uint32)
        w = np.zeros(max(e, 1), np.float64) if L.ref_graph_weighted(h) else None
        L.ref_graph_arrays(h, off, src, w.ctypes.data if w is not None else None, od)
        L.ref_graph_destroy(h)
        return CSC(n, off, src[:e], None if w is None else w[:e], od[:n])

    @classmethod
    def dumbbell(cls, k) -> CSC:
        n, e = C.c_uint64(), C.c_uint64()
        h = cls.lib().ref_generate_dumbbell(k, C.byref(n), C.byref(e))
        return cls._export(h, n.value, e.value)

    @classmethod
    def power_law(cls, nv, avg, ex, seed) -> CSC:
        n, e = C.c_uint64(), C.c_uint64()
        h = cls.lib().ref_generate_power_law(nv, avg, ex, seed, C.byref(n), C.byref(e))
        return cls._export(h, n.value, e.value)

    @classmethod
    def symmetrized(cls, g: CSC) -> CSC:
        n, e = C.c_uint64(), C.c_uint64()
        h0 = cls.graph(g)
        h = cls.lib().ref_symmetrized(h0, C.byref(n), C.byref(e))
        cls.free(h0)
        return cls._export(h, n.value, e.value)

    @classmethod
    def write_binary(cls, g: CSC, path: str):
        """The reference's GGCSR1 writer (graph.cpp:259-270)."""
        msg = C.create_string_buffer(256)
        h = cls.graph(g)
        rc = cls.lib().ref_write_binary(h, path.encode(), msg, 256)
        cls.free(h)
        if rc:
            raise RuntimeError(msg.value.decode())

    @classmethod
    def read_binary(cls, path: str) -> CSC:
        """The reference's GGCSR1 reader (graph.cpp:272-296); RuntimeError with
        its message on a bad file."""
        n, e = C.c_uint64(), C.c_uint64()
        msg = C.create_string_buffer(256)
        h = cls.lib().ref_read_binary(path.encode(), C.byref(n), C.byref(e), msg, 256)
        if not h:
            raise RuntimeError(msg.value.decode())
        return cls._export(h, n.value, e.value)

    @classmethod
    def sparsify(cls, g: CSC, sigma, seed):
        h = cls.graph(g)
        out = np.zeros(max(g.e, 1), np.uint8)
        rc = cls.lib().ref_sparsify(h, sigma, seed, out)
        cls.free(h)
        if rc:
            raise ValueError("sigma must be in [0,1]")
        return out[:g.e]

    @classmethod
    def run(cls, g, prog, scheme=ACCURATE, sigma=1.0, theta=0.0, alpha=1,
            max_iterations=100, seed=0, threads=1, handle=None, **pp) -> Result:
        L = cls.lib()
        params = _params(prog, **pp)
        cfg = _Config(scheme, sigma, theta, alpha, max_iterations, seed, threads)
        cap = max(1, min(max_iterations, 1 << 20))
        recs = (_RefRecord * cap)()
        summ = _RefSummary()
        props = _prop_shape(prog, g.n, pp.get("states", 2))
        msg = C.create_string_buffer(256)
        h = handle if handle is not None else cls.graph(g)
        rc = L.ref_run(h, prog, C.byref(params), C.byref(cfg), props.ctypes.data, recs, cap,
                       C.byref(summ), None, msg, 256)
        if handle is None:
            cls.free(h)
        k = int(min(summ.iterations_run, cap))
        return Result(rc, props, [int(recs[i].mode) for i in range(k)],
                      [int(recs[i].processed_edges) for i in range(k)],
                      [int(recs[i].active_vertices) for i in range(k)],
                      [float(recs[i].wall_seconds) for i in range(k)],
                      int(summ.iterations_run), int(summ.total_processed_edges),
                      int(summ.err_iteration), int(summ.err_vertex), msg.value.decode())

    @classmethod
    def metric(cls, which, approx, exact, k=0):
        r = C.c_double()
        a = np.ascontiguousarray(approx, np.float64); x = np.ascontiguousarray(exact, np.float64)
        if cls.lib().ref_metric(which, a, x, len(a), k, C.byref(r)):
            raise ValueError("reference metric raised")
        return r.value

    @classmethod
    def sweep_csv(cls, g: CSC, label, algo, schemes, sigmas, thetas, alphas, iterations,
                  repeats, seeds, sssp_source=0, sssp_graded=False, epsilon=-1.0) -> str:
        mask = sum({"sp": 1, "sms": 2, "gg": 4}[s] for s in schemes)
        buf = C.create_string_buffer(1 << 20)
        h = cls.graph(g)
        r = cls.lib().ref_sweep_csv(h, label.encode(), algo, mask,
                                    np.asarray(sigmas, np.float64), len(sigmas),
                                    np.asarray(thetas, np.float64), len(thetas),
                                    np.asarray(alphas, np.uint64), len(alphas), iterations,
                                    repeats, np.asarray(seeds, np.uint64), len(seeds),
                                    sssp_source, int(sssp_graded), epsilon, buf, 1 << 20)
        cls.free(h)
        if r < 0:
            raise RuntimeError("reference sweep failed")
        return buf.value.decode()
