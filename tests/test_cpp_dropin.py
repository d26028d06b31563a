"""The C++ drop-in boundary (include/ggb_gg.hpp).

* GPU: tests/cpp/bin/test_dropin runs the reference gg::run and ggb::run on the
  same gg:: objects and compares reports and exceptions (see its header).
* CPU: a VertexProgram with no device entry must not compile (no fallback),
  and the four reference programs must; needs the reference headers, so it
  runs only where /root/reference exists.
"""
from __future__ import annotations

import os
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "bin", "test_dropin")
REF_INC = "/root/reference/proj/core/include"


@pytest.mark.gpu
def test_dropin_matches_reference_engine():
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/bin/test_dropin not built (needs the reference headers at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    print(r.stdout[-2000:], r.stderr[-4000:])
    assert r.returncode == 0, r.stderr[-4000:]
    assert ", 0 failed" in r.stdout


def _compile(src: str):
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "t.cpp")
        open(p, "w").write(src)
        return subprocess.run(["/usr/bin/g++", "-std=c++20", "-fsyntax-only", "-I" + REF_INC,
                               "-I" + os.path.join(ROOT, "include"), p],
                              capture_output=True, text=True, timeout=120)


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers absent")
def test_reference_programs_have_device_entries():
    r = _compile("""
#include "ggb_gg.hpp"
void f(const gg::Graph& g, const gg::EngineConfig& c) {
    gg::RunReport<double> a = ggb::run(g, gg::pagerank_spec(), c);
    gg::RunReport<double> b = ggb::run(g, gg::sssp_spec(0, true), c);
    gg::RunReport<std::uint32_t> w = ggb::run(g, gg::wcc_spec(), c);
    gg::RunReport<std::vector<double>> p = ggb::run(g, gg::bp_spec(2), c);
}
""")
    assert r.returncode == 0, r.stderr


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers absent")
def test_program_without_device_entry_is_a_compile_error():
    r = _compile("""
#include "ggb_gg.hpp"
struct Custom : gg::PageRankProgram {};   // a new VertexProgram, no device program
void f(const gg::Graph& g, const gg::EngineConfig& c) { ggb::run(g, Custom{}, c); }
""")
    assert r.returncode != 0
    assert "no compiled device program" in r.stderr
