"""The oracle's lock-step mask comparison (og_run_ex) and its thread
invariance, on CPU (no device): the machinery the GPU mask-parity tests
(tests/parity.py) rely on.

* og_run over OpenMP threads equals the sequential run bit for bit
  (test_engine.cpp:161-182 is the reference's own thread-invariance case).
* Fed its own superstep flags as the "device" flags, the lock-step run
  adopts nothing and equals the plain run.
* A flipped flag on an edge whose influence equals theta exactly (inside the
  rounding band) is adopted and counted; a flipped flag far from theta is a
  real mismatch, counted, and not adopted.
"""
import numpy as np
import pytest

from oracle.oracle import BP, GG, PR, SMS, SSSP, WCC, Oracle
from tests.parity import NEAR_UNIT


def _pack(flags):
    return np.packbits(flags.astype(np.uint8), bitorder="little").view(np.uint8)


def _words(flags):
    b = _pack(flags)
    pad = (-len(b)) % 4
    return np.concatenate([b, np.zeros(pad, np.uint8)]).view(np.uint32)


CASES = [(PR, {}), (SSSP, dict(graded=True)), (WCC, {}), (BP, dict(states=3, coupling=0.7))]


@pytest.mark.parametrize("prog,pp", CASES)
def test_threads_bitwise_invariant(prog, pp):
    g = Oracle.power_law(3000, 9.0, 2.1, 4)
    if prog == WCC:
        g = Oracle.symmetrized(g)
    kw = dict(scheme=GG, sigma=0.5, theta=0.05, alpha=2, max_iterations=20, seed=3, want_flags=True)
    a = Oracle.run(g, prog, threads=1, **kw, **pp)
    b = Oracle.run(g, prog, threads=4, **kw, **pp)
    assert a.status == b.status == 0
    assert np.array_equal(a.props.view(np.uint8), b.props.view(np.uint8))
    assert a.processed_edges == b.processed_edges and a.active_vertices == b.active_vertices
    assert np.array_equal(a.flags, b.flags)


def _superstep_flags(g, prog, kw, pp):
    plain = Oracle.run(g, prog, want_flags=True, **kw, **pp)
    its = [i + 1 for i, m in enumerate(plain.modes) if m == 2]
    dev = []
    for t in its:
        k2 = dict(kw, max_iterations=t)
        dev.append(_words(Oracle.run(g, prog, want_flags=True, **k2, **pp).flags))
    return plain, its, dev


@pytest.mark.parametrize("prog,pp", CASES)
def test_lockstep_own_flags_adopts_nothing(prog, pp):
    g = Oracle.power_law(2000, 8.0, 2.1, 5)
    kw = dict(scheme=GG, sigma=0.5, theta=0.05, alpha=2, max_iterations=15, seed=5, threads=2)
    plain, its, dev = _superstep_flags(g, prog, kw, pp)
    assert its
    r = Oracle.run(g, prog, want_flags=True, device_flags=dev, tol_unit=NEAR_UNIT[prog], **kw, **pp)
    assert [s["adopted"] for s in r.lockstep] == [0] * len(its)
    assert [s["real"] for s in r.lockstep] == [0] * len(its)
    assert all(s["compared"] for s in r.lockstep)
    assert np.array_equal(r.flags, plain.flags)
    assert r.processed_edges == plain.processed_edges
    assert np.array_equal(r.props.view(np.uint8), plain.props.view(np.uint8))


def test_lockstep_adopts_tie_and_counts_real_flip():
    """PR, sms scheme (one superstep at t = alpha + 1 = 3)."""
    g = Oracle.power_law(1500, 10.0, 2.1, 8)
    base = dict(scheme=SMS, sigma=0.5, alpha=2, seed=8, threads=2)
    # influences at the superstep, from the properties after iteration 2
    prev = Oracle.run(g, PR, theta=0.0, max_iterations=2, **base).props
    infl = Oracle.influences(g, PR, prev, threads=2)
    v = int(np.argmax(np.diff(g.off.astype(np.int64))))  # the hub: processed in the superstep
    e0, e1 = int(g.off[v]), int(g.off[v + 1])
    # an edge whose influence is an exact tie with theta: estatus(infl > theta) is false
    e_tie = e0 + 7
    theta = float(infl[e_tie])
    kw = dict(base, theta=theta, max_iterations=3)
    own = Oracle.run(g, PR, want_flags=True, **kw)
    assert own.flags[e_tie] == 0
    # a kept edge far from theta (influence 1: the first edge of the list)
    e_far = e0
    assert infl[e_far] == 1.0 and own.flags[e_far] == 1
    dev = own.flags.copy()
    dev[e_tie] = 1   # inside the band: adopted
    dev[e_far] = 0   # outside the band: real mismatch, not adopted
    r = Oracle.run(g, PR, want_flags=True, device_flags=[_words(dev)], tol_unit=NEAR_UNIT[PR], **kw)
    (s,) = r.lockstep
    assert s["adopted"] == 1 and s["real"] == 1 and s["near"] >= 1
    assert r.flags[e_tie] == 1 and r.flags[e_far] == 1
    assert e1 > e_tie
    # the min programs have no band: the same flip on an SSSP tie is real
    assert NEAR_UNIT[SSSP] == 0.0 and NEAR_UNIT[WCC] == 0.0
