"""CPU tests of the C-ABI boundary: the library loads, exports every symbol that
include/spin.h declares, and its host-only logic (chunk tables, region radius,
cosines) agrees with the independent oracle and the goldens.  No compute calls."""
import ctypes
import json
import math
import os
import re

import numpy as np
import pytest

from oracle import spin_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "spin.h")


def _declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(spin_[A-Za-z_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    from paper_1811_00901_b200 import spin
    lib = ctypes.CDLL(spin.LIB_PATH)
    names = _declared()
    assert len(names) >= 10
    for n in names:
        assert hasattr(lib, n), f"libspin.so does not export {n}"
    assert set(names) == set(spin.EXPORTS)
    assert spin.abi_version() == 6


def test_binding_has_no_cpu_fallback():
    """The product package must not import the oracle or any CPU implementation."""
    pkg = os.path.join(ROOT, "paper_1811_00901_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                src = open(os.path.join(dp, f)).read()
                assert "from oracle" not in src and "import oracle" not in src, f


@pytest.mark.parametrize("kind", [O.STATIC, O.SS, O.GSS, O.FAC])
def test_chunk_sequence_matches_oracle(kind):
    from paper_1811_00901_b200 import spin
    rng = np.random.default_rng(kind)
    for _ in range(200):
        n = int(rng.integers(0, 30000))
        P = int(rng.integers(1, 600))
        if kind == O.SS:
            n = min(n, 3000)
        g = int(rng.integers(1, 4))
        f = int(rng.integers(1, 4))
        assert spin.chunk_sequence(kind, n, P, gss_min_chunk=g, fac_divisor=f) == \
            O.chunk_bounds(kind, n, P, gss_min_chunk=g, fac_divisor=f)


def test_weighted_factoring_matches_oracle():
    from paper_1811_00901_b200 import spin
    rng = np.random.default_rng(11)
    for _ in range(200):
        n = int(rng.integers(0, 30000))
        P = int(rng.integers(1, 600))
        f = int(rng.integers(1, 4))
        S = int(rng.integers(0, P + 1))
        sd = float(np.float32(rng.uniform(1.0, 8.0)))
        assert spin.chunk_sequence("WF", n, P, fac_divisor=f, slow_ctas=S, slowdown=sd) == \
            O.chunk_bounds(O.WF, n, P, fac_divisor=f, slow=S, slowdown=sd)
    with pytest.raises(spin.SpinError):
        spin.chunk_sequence("AWF", 100, 4)   # measured weights: no static trace


def test_chunk_goldens_through_abi():
    from paper_1811_00901_b200 import spin
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "chunks.json")))
    d = lambda b: list(np.diff(b))
    assert d(spin.chunk_sequence("GSS", 100, 4)) == g["GSS_100_4"]
    assert d(spin.chunk_sequence("FAC", 100, 4)) == g["FAC_100_4"]
    assert d(spin.chunk_sequence("STATIC", 10, 4)) == g["STATIC_10_4"]
    assert d(spin.chunk_sequence("STATIC", 7, 7)) == g["STATIC_7_7"]
    assert len(spin.chunk_sequence("SS", 100, 4)) == 101
    assert spin.chunk_sequence("GSS", 0, 4) == [0]


def test_chunk_sequence_errors():
    from paper_1811_00901_b200 import spin
    with pytest.raises(spin.SpinError):
        spin.chunk_sequence("GSS", 10, 0)
    with pytest.raises(spin.SpinError):
        spin.chunk_sequence(7, 10, 2)


@pytest.mark.parametrize("mode,flags", [(0, 0), (0, O.F_FLOOR_BINS), (1, 0),
                                        (0, O.F_LITERAL_HALF_WIDTH), (1, O.F_LITERAL_HALF_WIDTH)])
def test_region_radius_matches_oracle(mode, flags):
    from paper_1811_00901_b200 import spin
    for W in (1, 2, 5, 8, 16, 24, 32, 64):
        for b in (0.005, 0.02, 0.1, 1.0):
            if mode == 1 and W < 2:
                continue
            a = spin.region_radius(W, b, mode, flags)
            o = O.region_radius(W, b, mode, flags)
            assert abs(a - o) <= 1e-9 * o


def test_cos_from_degrees_exact():
    from paper_1811_00901_b200 import spin
    assert spin.cos_from_degrees(0) == 1.0
    assert spin.cos_from_degrees(60) == 0.5
    assert spin.cos_from_degrees(90) == 0.0
    assert spin.cos_from_degrees(120) == -0.5
    assert spin.cos_from_degrees(180) == -math.inf
    assert spin.cos_from_degrees(360) == -math.inf
    assert abs(spin.cos_from_degrees(45) - math.sqrt(0.5)) < 1e-15


def test_header_documents_every_entry_point():
    txt = open(HEADER).read()
    for n in _declared():
        # each declaration is preceded by a comment block naming it or its family
        assert n in txt
    assert "PAPER.md:146-182" in txt and "PAPER.md:286-319" in txt


def test_binding_refuses_bad_clouds_before_any_cuda_call():
    """spin.py marshals only contiguous float32 [N, 3] clouds; anything else is a
    ValueError raised before the C ABI is called (no silent reinterpretation)."""
    from paper_1811_00901_b200 import spin
    P = np.zeros((10, 3), np.float32)
    for bad in (P.astype(np.float64), P[:, :2], np.asfortranarray(np.zeros((10, 3), np.float32))[::2]):
        with pytest.raises(ValueError):
            spin.SpinEngine(bad, P)
    with pytest.raises(ValueError):
        spin.SpinEngine(P, np.zeros((9, 3), np.float32))


def test_oracle_sources_are_independent_of_the_product():
    """The C++ oracle includes nothing from the product tree and the product never names it."""
    src = open(os.path.join(ROOT, "oracle", "spin_oracle.cpp")).read()
    assert "spin.h" not in src and "spin_internal" not in src and "csrc" not in src
    for inc in re.findall(r'#include\s+[<"]([^>"]+)[>"]', src):
        assert "/" not in inc and not inc.startswith("spin"), inc
