"""Generates the golden fixtures in tests/golden/ FROM THE REFERENCE ITSELF.

Runs the unmodified GraphGuess reference (oracle/_ref/libggref.so, compiled
from /root/reference by oracle/Makefile) on small seeded inputs and stores
its outputs, so the CPU oracle (and through it the device engine) can be
pinned on boxes where /root/reference does not exist.

    python tests/golden/make_golden.py      # needs oracle/_ref/libggref.so
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import BP, BP_EDGE, PR, SSSP, WCC, Oracle, Reference  # noqa: E402

SCHEMES = {"accurate": 0, "sp": 1, "sms": 2, "gg": 3}


def graphs():
    """Seeded small inputs: the reference's own generators / test fixtures."""
    out = {}
    for k in (2, 3, 4, 8):
        out[f"dumbbell{k}"] = ("dumbbell", dict(k=k))
    for s in (1, 2, 3):
        out[f"powerlaw300_s{s}"] = ("power_law", dict(n=300, avg=6.0, ex=2.2, seed=s))
        out[f"random200w_s{s}"] = ("random", dict(n=200, m=1500, seed=s, weighted=True))
    return out


def build(kind, p):
    if kind == "dumbbell":
        return Reference.dumbbell(p["k"])
    if kind == "power_law":
        return Reference.power_law(p["n"], p["avg"], p["ex"], p["seed"])
    if kind == "random":
        return Oracle.random_graph(p["n"], p["m"], p["seed"], p["weighted"])  # test_support.hpp fixture
    if kind == "rmat":
        return Oracle.rmat(p["scale"], p["ef"], p["seed"])
    raise ValueError(kind)


def f64hex(a):
    return [float(x).hex() for x in np.asarray(a, np.float64).reshape(-1)]


def main():
    if not Reference.available():
        sys.exit("oracle/_ref/libggref.so missing: run `make -C oracle ref` first")
    fixtures = {"graphs": {}, "runs": []}
    gs = graphs()
    for name, (kind, p) in gs.items():
        g = build(kind, p)
        fixtures["graphs"][name] = {"kind": kind, "params": p, "n": g.n, "e": g.e,
                                    "src_sum": int(g.src.astype(np.int64).sum()),
                                    "off_sum": int(g.off.astype(np.int64).sum())}
        progs = [(PR, {}), (BP, {}), (BP, dict(states=3, coupling=0.7))]
        if g.w is not None:
            progs += [(SSSP, {}), (SSSP, dict(graded=True))]
        else:
            progs += [(SSSP, {})]
        for prog, pp in progs + [(WCC, {})]:
            graph = Reference.symmetrized(g) if prog == WCC else g
            for scheme in ("accurate", "sp", "sms", "gg"):
                cfg = dict(scheme=SCHEMES[scheme], sigma=0.5 if scheme != "accurate" else 1.0,
                           theta=0.1, alpha=3, max_iterations=25, seed=7)
                r = Reference.run(graph, prog, **cfg, **pp)
                props = r.props.astype(np.float64) if prog != WCC else r.props
                fixtures["runs"].append({
                    "graph": name, "prog": prog, "params": pp, "config": cfg,
                    "status": r.status, "iterations_run": r.iterations_run,
                    "modes": r.modes, "processed_edges": r.processed_edges,
                    "active_vertices": r.active_vertices,
                    "props": [int(x) for x in props] if prog == WCC else f64hex(props),
                })
    # BASELINE-C4-style edge BP (new program type handed to the reference gg::run)
    g = Oracle.rmat(9, 16, 4)
    c = Oracle.bp_couplings(g.e, 4)
    dst = np.repeat(np.arange(g.n), np.diff(g.off.astype(np.int64)))
    gw = Oracle.build_graph(g.n, g.src, dst, c.astype(np.float64))
    pri = Oracle.bp_priors(g.n, 4)
    for scheme in ("accurate", "gg"):
        cfg = dict(scheme=SCHEMES[scheme], sigma=0.5, theta=0.01, alpha=4, max_iterations=30, seed=4)
        r = Reference.run(gw, BP_EDGE, prior_table=pri, **cfg)
        fixtures["runs"].append({"graph": "rmat9_s4_bpedge", "prog": BP_EDGE, "params": {},
                                 "config": cfg, "status": r.status,
                                 "iterations_run": r.iterations_run, "modes": r.modes,
                                 "processed_edges": r.processed_edges,
                                 "active_vertices": r.active_vertices, "props": f64hex(r.props)})
    fixtures["graphs"]["rmat9_s4_bpedge"] = {"kind": "rmat_bpedge", "params": dict(scale=9, ef=16, seed=4),
                                             "n": gw.n, "e": gw.e}
    # sparsify masks (engine.cpp:63-75)
    h = Reference.sparsify(Oracle.random_graph(200, 100000, 4), 0.5, 3)
    fixtures["sparsify_e100000_s3_popcount"] = int(h.sum())
    fixtures["sparsify_e2000_prefix"] = {
        "sigma": 0.3, "seed": 5,
        "bits": "".join(str(int(b)) for b in Reference.sparsify(Oracle.random_graph(60, 2000, 8), 0.3, 5))}
    with open(os.path.join(HERE, "reference_runs.json"), "w") as f:
        json.dump(fixtures, f, separators=(",", ":"))
    # the reference's sweep CSV for the dumbbell plan (test_bench.cpp:16-29)
    csv = Reference.sweep_csv(Reference.dumbbell(4), "gen:dumbbell:4", 2, ["sp", "gg"], [0.4, 0.8],
                              [0.5], [2], 16, 1, [1, 2])
    with open(os.path.join(HERE, "dumbbell4_sweep.csv"), "w") as f:
        f.write(csv)
    print(f"wrote {len(fixtures['runs'])} reference runs")


if __name__ == "__main__":
    main()
