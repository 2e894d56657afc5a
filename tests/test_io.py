"""CPU tests of host-side ingestion through the C ABI:
spin_read_xyzn, spin_read_off, spin_vertex_normals.  No GPU needed.  Pins: the SPEC's
worked cases (axis normal normalised, zero normal rejected, single triangle),
symmetry (regular tetrahedron / octahedron vertex normals point away from the centre),
and a write/read round trip of a synthetic cloud."""
import os

import numpy as np
import pytest

from synth import clouds


@pytest.fixture(scope="module")
def spin():
    from paper_1811_00901_b200 import spin as s
    return s


def _write(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def test_xyzn_normalises_and_keeps_order(spin, tmp_path):
    p = _write(tmp_path, "a.xyzn", "# comment\n0 0 0 0 0 2\n\n1 2 3  3 0 4  # tail\n")
    P, N = spin.read_xyzn(p)
    np.testing.assert_array_equal(P, [[0, 0, 0], [1, 2, 3]])
    np.testing.assert_array_equal(N, np.float32([[0, 0, 1], [0.6, 0, 0.8]]))


@pytest.mark.parametrize("text,needle", [("0 0 0 0 0 0\n", "zero normal"),
                                         ("0 0 0 0 0\n", ":1:"),
                                         ("1 1 1 0 0 1\n0 0 x 0 0 1\n", ":2:"),
                                         ("# only a comment\n", "empty"),
                                         ("0 0 0 0 0 1 7\n", ":1:"),
                                         ("0 0 inf 0 0 1\n", "non-finite")])
def test_xyzn_errors(spin, tmp_path, text, needle):
    p = _write(tmp_path, "bad.xyzn", text)
    with pytest.raises(spin.SpinError) as e:
        spin.read_xyzn(p)
    assert needle in str(e.value)


def test_xyzn_round_trip_synthetic(spin, tmp_path):
    P, N = clouds.bumpy_sphere(500, 3)
    p = str(tmp_path / "c.xyzn")
    np.savetxt(p, np.hstack([P, N]).astype(np.float64), fmt="%.9g")
    P2, N2 = spin.read_xyzn(p)
    np.testing.assert_array_equal(P2, P)                   # %.9g round-trips fp32 exactly
    np.testing.assert_allclose(np.linalg.norm(N2.astype(np.float64), axis=1), 1.0, atol=1e-7)
    np.testing.assert_allclose(N2, N, atol=2e-7)           # generator normals are unit already


def _off(V, F):
    lines = ["OFF", f"{len(V)} {len(F)} 0"]
    lines += [" ".join(repr(float(c)) for c in v) for v in V]
    lines += ["3 " + " ".join(str(int(i)) for i in f) for f in F]
    return "\n".join(lines) + "\n"


def test_single_triangle_normal(spin, tmp_path):
    V = np.float32([[0, 0, 0], [1, 0, 0], [0, 1, 0]])
    p = _write(tmp_path, "t.off", _off(V, [[0, 1, 2]]))
    V2, F2 = spin.read_off(p)
    np.testing.assert_array_equal(V2, V)
    np.testing.assert_array_equal(F2, [[0, 1, 2]])
    np.testing.assert_array_equal(spin.vertex_normals(V2, F2), np.float32([[0, 0, 1]] * 3))
    # a second coplanar triangle leaves every normal unchanged
    V4 = np.float32([[0, 0, 0], [1, 0, 0], [0, 1, 0], [1, 1, 0]])
    np.testing.assert_array_equal(spin.vertex_normals(V4, [[0, 1, 2], [1, 3, 2]]),
                                  np.float32([[0, 0, 1]] * 4))


@pytest.mark.parametrize("solid", ["tetrahedron", "octahedron"])
def test_symmetric_solids_point_outward(spin, tmp_path, solid):
    """Each vertex of a regular solid meets congruent faces symmetrically, so its
    area-weighted normal is the direction from the centre (outward winding)."""
    if solid == "tetrahedron":
        V = np.float32([[1, 1, 1], [1, -1, -1], [-1, 1, -1], [-1, -1, 1]])
        F = [[0, 1, 2], [0, 3, 1], [0, 2, 3], [1, 3, 2]]
    else:
        V = np.float32([[1, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1], [0, 0, -1]])
        F = [[0, 2, 4], [2, 1, 4], [1, 3, 4], [3, 0, 4], [2, 0, 5], [1, 2, 5], [3, 1, 5], [0, 3, 5]]
    p = _write(tmp_path, "s.off", _off(V, F))
    V2, F2 = spin.read_off(p)
    N = spin.vertex_normals(V2, F2)
    want = V / np.linalg.norm(V, axis=1, keepdims=True)
    np.testing.assert_allclose(N, want, atol=1e-7)
    Pc, Nc = spin.load_mesh_cloud(p)
    np.testing.assert_array_equal(Nc, N)


def test_off_errors(spin, tmp_path):
    with pytest.raises(spin.SpinError, match="OFF header"):
        spin.read_off(_write(tmp_path, "a.off", "PLY\n"))
    with pytest.raises(spin.SpinError, match="out of range"):
        spin.read_off(_write(tmp_path, "b.off", "OFF\n3 1 0\n0 0 0\n1 0 0\n0 1 0\n3 0 1 3\n"))
    with pytest.raises(spin.SpinError, match="triangle"):
        spin.read_off(_write(tmp_path, "c.off", "OFF\n4 1 0\n0 0 0\n1 0 0\n0 1 0\n1 1 0\n4 0 1 3 2\n"))
    V = np.float32([[0, 0, 0], [1, 0, 0], [0, 1, 0], [5, 5, 5]])
    with pytest.raises(spin.SpinError, match="no incident face"):
        spin.vertex_normals(V, [[0, 1, 2]])
    with pytest.raises(spin.SpinError, match="outside"):
        spin.vertex_normals(V, [[0, 1, 7]])
