"""The C-ABI boundary on CPU: libggb.so loads, exports every symbol that
include/ggb.h declares, its host-only entry points behave like the
reference (engine.cpp / metrics.cpp), and compute entries fail loudly
without an sm_100 GPU (no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from oracle.oracle import ACCURATE, GG, SMS, SP, Oracle
from tests.conftest import ROOT, has_gpu

HEADER = os.path.join(ROOT, "include", "ggb.h")
LIB = os.path.join(ROOT, "paper_2104_10039_b200", "libggb.so")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(gg_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported():
    syms = declared_symbols()
    assert len(syms) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r" T (gg_[a-z0-9_]+)$", out, re.M))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    lib = ctypes.CDLL(LIB)
    for s in syms:
        assert hasattr(lib, s)


def test_python_binding_lists_every_export():
    from paper_2104_10039_b200 import _lib
    assert sorted(_lib.EXPORTS) == declared_symbols()


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_abi_version_and_status_strings(ggb):
    from paper_2104_10039_b200 import _lib
    lib = _lib.lib()
    assert lib.gg_abi_version() == 5
    assert _lib.status_string(_lib.GG_INVALID_PROPERTY) == "invalid property"
    assert _lib.status_string(99) == "unknown status"


def test_mode_and_schedule_match_reference(ggb):  # engine.cpp:77-107
    for scheme in (ACCURATE, SP, SMS, GG):
        for alpha in (1, 2, 3, 5):
            for t in range(1, 30):
                assert int(ggb.mode_for(scheme, t, alpha)) == Oracle.mode_for(scheme, t, alpha)
            for mx in (1, 3, 10, 29):
                assert ggb.select_superstep_iterations(alpha, mx, scheme) == \
                    Oracle.supersteps(alpha, mx, scheme)
    assert ggb.select_superstep_iterations(2, 10, "gg") == [3, 6, 9]


def test_validate_messages(ggb):  # engine.cpp:45-61
    for kw, field in ((dict(sigma=1.5), "sigma"), (dict(sigma=-0.1), "sigma"),
                      (dict(theta=-1.0), "theta"), (dict(alpha=0), "alpha"),
                      (dict(max_iterations=0), "max_iterations"), (dict(threads=0), "threads")):
        with pytest.raises(ValueError, match=field):
            ggb.validate(ggb.EngineConfig(**kw))
    ggb.validate(ggb.EngineConfig("gg", 0.5, 0.1, 3, 10, 1))
    with pytest.raises(ValueError, match="unknown scheme"):
        ggb.EngineConfig("bogus").c()


def test_factory_domain_checks(ggb):  # algorithms.cpp:71-98
    for args in ((0.0, 1e-7), (1.0, 1e-7), (0.85, 0.0)):
        with pytest.raises(ValueError):
            ggb.pagerank_spec(*args)
    for args in ((1, 0.8, 1e-6), (2, 0.0, 1e-6), (2, 1.0, 1e-6), (2, 0.8, 0.0)):
        with pytest.raises(ValueError):
            ggb.bp_spec(*args)


def test_host_metrics_match_oracle(ggb):  # metrics.cpp
    rng = np.random.default_rng(3)
    for _ in range(50):
        a, e = rng.random(60), rng.random(60)
        for k in (1, 5, 60):
            assert ggb.topk_error(a, e, k).error == Oracle.topk_error(a, e, k)
        assert ggb.relative_error(a, e).error == Oracle.relative_error(a, e)
        s = np.sort(rng.random(60))
        assert ggb.stretch_error(s + 0.1, s).error == Oracle.stretch_error(s + 0.1, s)
    with pytest.raises(ValueError):
        ggb.topk_error([1, 2], [1, 2], 3)
    with pytest.raises(RuntimeError):
        ggb.stretch_error([0.0, 1.0], [0.0, 2.0])
    r = ggb.topk_error([9, 8, 7, 1, 0], [9, 8, 1, 7, 0], 3)
    assert abs(r.accuracy - 66.6667) < 1e-3


def test_partition_plan_is_edge_balanced_and_aligned(ggb):
    g = Oracle.rmat(14, 16, 3)
    graph = ggb.Graph(g.n, g.off, g.src)
    for nranks in (1, 2, 4, 8):
        b = ggb.partition_plan(graph, nranks)
        assert b[0] == 0 and b[-1] == g.n and np.all(np.diff(b.astype(np.int64)) >= 0)
        assert all(int(x) % 32 == 0 for x in b[:-1])
        edges = np.diff(g.off[b.astype(np.int64)].astype(np.int64))
        assert edges.max() <= g.e / nranks + 32 * int(np.diff(g.off.astype(np.int64)).max())


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU failure path")
def test_compute_entries_fail_loudly_without_gpu(ggb):
    g = Oracle.dumbbell(2)
    with pytest.raises(ggb.GgbError, match="CUDA"):
        ggb.run(ggb.Graph(g.n, g.off, g.src), ggb.pagerank_spec(), ggb.EngineConfig())
