"""The host-side helpers behind ``import icemorph`` (paper_2107_13887_b200/
host_tools.py: generators, VTK / displacement files, report writers) against
the reference's own implementations (oracle/_ref, generators.cpp and
mesh_io.cpp), bit for bit / byte for byte.  CPU only."""
import ctypes as C

import numpy as np
import pytest

import icemorph as im

_d, _sz = C.c_double, C.c_size_t
_pd, _psz = C.POINTER(C.c_double), C.POINTER(C.c_size_t)


def _ref_mesh(ref, n, m):
    f = ref.lib.ref_gen_airfoil_mesh
    f.argtypes = [_d, _sz, _sz, _pd, _psz, _psz, _psz]
    nodes = np.zeros((n * (m + 1), 3))
    quads = np.zeros((n * m, 4), np.uint64)
    air, far = np.zeros(n, np.uint64), np.zeros(n, np.uint64)
    ref._check(f(1.0, n, m, nodes.ctypes.data_as(_pd), quads.ctypes.data_as(_psz),
                 air.ctypes.data_as(_psz), far.ctypes.data_as(_psz)))
    return nodes, quads, air, far


@pytest.mark.parametrize("n,m", [(64, 8), (128, 12), (400, 250)])
def test_airfoil_mesh_matches_reference(ref, n, m):
    nodes, quads, air, far = _ref_mesh(ref, n, m)
    mesh = im.gen_airfoil_mesh(1.0, n, m)
    assert np.array_equal(np.array(mesh.nodes()), nodes)
    k, o, c = mesh._elements
    assert np.array_equal(c.reshape(-1, 4), quads) and np.all(k == 2)
    assert mesh.marker_nodes("airfoil") == air.tolist()
    assert mesh.marker_nodes("farfield") == far.tolist()


@pytest.mark.parametrize("which,params", [(0, (0.01, 15.0, 0.0, 0)), (0, (0.03, 4.0, 0.0, 0)),
                                          (1, (0.0, 0.02, 0.05, 2)), (1, (0.1, 0.03, 0.02, 3))])
def test_displacement_generators_match_reference(ref, which, params):
    n, m = 128, 12
    f = ref.lib.ref_gen_field
    f.argtypes = [_d, _sz, _sz, C.c_int, _d, _d, _d, _sz, _psz, _pd, _psz]
    idx, disp, cnt = np.zeros(n, np.uint64), np.zeros((n, 3)), _sz()
    ref._check(f(1.0, n, m, which, params[0], params[1], params[2], params[3],
                 idx.ctypes.data_as(_psz), disp.ctypes.data_as(_pd), C.byref(cnt)))
    mesh = im.gen_airfoil_mesh(1.0, n, m)
    if which == 0:
        g = im.gen_sinusoidal_displacement(mesh, "airfoil", "airfoil", params[0], params[1])
    else:
        g = im.gen_ice_bump(mesh, "airfoil", params[0], params[1], params[2], params[3])
    e = g.entries()
    assert sorted(e) == idx[:cnt.value].tolist()
    assert np.array_equal(np.array([e[int(i)] for i in idx[:cnt.value]]), disp[:cnt.value])


def test_writers_match_reference_bytes(ref, tmp_path):
    # the reference's ostream writers crash once numpy is loaded in the same
    # process, so they run in a numpy-free subprocess
    import subprocess
    import sys

    import pyoracle

    rv, rd = tmp_path / "ref.vtk", tmp_path / "ref.disp"
    code = ("import ctypes as C, sys; L = C.CDLL(sys.argv[1]); f = L.ref_write_airfoil_files; "
            "f.argtypes = [C.c_double, C.c_size_t, C.c_size_t, C.c_char_p, C.c_char_p]; "
            "sys.exit(f(1.0, 64, 8, sys.argv[2].encode(), sys.argv[3].encode()))")
    r = subprocess.run([sys.executable, "-c", code, pyoracle.LIBS["ref"], str(rv), str(rd)],
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    mesh = im.gen_airfoil_mesh(1.0, 64, 8)
    im.write_vtk(mesh, str(tmp_path / "b.vtk"))
    im.write_displacements(im.gen_ice_bump(mesh, "airfoil"), mesh.dim, str(tmp_path / "b.disp"))
    assert (tmp_path / "b.vtk").read_bytes() == rv.read_bytes()
    assert (tmp_path / "b.disp").read_bytes() == rd.read_bytes()
    back = im.read_displacements(str(rd), mesh, "airfoil")
    assert back.entries() == im.gen_ice_bump(mesh, "airfoil").entries()


def test_errors_match_reference_messages(tmp_path):
    mesh = im.gen_airfoil_mesh(1.0, 64, 8)
    with pytest.raises(ValueError, match="mesh has no marker named 'nope'"):
        im.gen_sinusoidal_displacement(mesh, "nope")
    with pytest.raises(ValueError, match="circumferential count must be even"):
        im.gen_airfoil_mesh(1.0, 65, 8)
    p = tmp_path / "bad.disp"
    p.write_text("3 0.1\n")
    with pytest.raises(RuntimeError, match=":1: expected `node dx dy`, got 2 tokens"):
        im.read_displacements(str(p), mesh, "airfoil")
    p.write_text("# comment\n9999 0.1 0.2\n")
    with pytest.raises(RuntimeError, match=":2: node 9999 is not on marker 'airfoil'"):
        im.read_displacements(str(p), mesh, "airfoil")
