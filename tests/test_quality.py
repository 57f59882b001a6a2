"""signed_measures / count_inverted (quality.cpp:100-148) and the report's
inverted_elements (pipeline.cpp:101).

CPU tests pin the plain-C oracle against the reference's own quality tests
(tests/test_quality.cpp:68-128) and against the reference on random meshes;
GPU tests hold the CUDA product (im_signed_measures / im_count_inverted /
im_deform with elements) bit-exact to the oracle: measures compared as bit
patterns, counts exactly."""
import math

import numpy as np
import pytest

import meshes as M
from paper_2107_13887_b200 import capi, workloads as W


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def five_tet_hex(p):
    """tests/oracles.cpp:109-120, the reference test's independent hex oracle."""
    def tet(a, b, c, d):
        return np.dot(p[b] - p[a], np.cross(p[c] - p[a], p[d] - p[a])) / 6.0
    return tet(0, 1, 3, 4) + tet(2, 3, 1, 6) + tet(5, 4, 6, 1) + tet(7, 6, 4, 3) + tet(1, 3, 4, 6)


# ---- oracle (CPU) ------------------------------------------------------------------
def test_canonical_triangle(port):  # test_quality.cpp:68-78
    nodes = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], float)
    m, inv = port.signed_measures(nodes, 2, M.csr([(M.TRI, [0, 1, 2]), (M.TRI, [0, 2, 1])]))
    assert m[0] == 0.5 and m[1] == -0.5 and inv == 1


def test_hex_prism_pyramid(port):  # test_quality.cpp:80-113
    nodes, el = M.box_grid(1, 1, 1)
    m, _ = port.signed_measures(nodes, 3, M.csr(el))
    assert m[0] == pytest.approx(1.0, rel=1e-14)
    skew = nodes + np.outer(nodes[:, 2], [0.25, 0.1, 0.0])
    ms, _ = port.signed_measures(skew, 3, M.csr(el))
    assert ms[0] == pytest.approx(five_tet_hex(skew[el[0][1]]), rel=1e-13)
    pn = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [1, 0, 1], [0, 1, 1]], float)
    mp, _ = port.signed_measures(pn, 3, M.csr([(M.PRISM, list(range(6)))]))
    assert mp[0] == pytest.approx(0.5, rel=1e-14)
    yn = np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0], [0.5, 0.5, 1.0]])
    my, _ = port.signed_measures(yn, 3, M.csr([(M.PYRAMID, list(range(5)))]))
    assert my[0] == pytest.approx(1.0 / 3.0, rel=1e-14)


def test_broken_hex_counted(port):  # test_quality.cpp:115-128
    nodes, el = M.box_grid(3, 2, 2)
    good, inv0 = port.signed_measures(nodes, 3, M.csr(el))
    n = el[0][1]
    el[0] = (M.HEX, n[4:] + n[:4])
    bad, inv1 = port.signed_measures(nodes, 3, M.csr(el))
    assert inv0 == 0 and inv1 == 1
    assert bad[0] == pytest.approx(-good[0], rel=1e-13)


def test_port_matches_golden_quality(port, golden):
    e = (golden["q_kinds"], golden["q_offsets"], golden["q_conn"])
    m, inv = port.signed_measures(golden["q_nodes"], 3, e)
    assert np.array_equal(bits(m), bits(golden["q_measures"]))
    assert inv == int(golden["q_inverted"])


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_port_matches_reference_quality(port, ref, seed):
    nodes, e = M.random_mixed(np.random.default_rng(seed), 200, 2000)
    mp, ip = port.signed_measures(nodes, 3, e)
    mr, ir = ref.signed_measures(nodes, 3, e)
    assert np.array_equal(bits(mp), bits(mr)) and ip == ir


def _sheared_quad_grid():  # test_quality.cpp:36-44
    nodes, el, _ = M.quad_grid(5, 4, 2.0, 1.0)
    nodes[8, 0] += 0.13
    nodes[8, 1] += 0.07
    return nodes, el


def test_orthogonality_kats(port):  # test_quality.cpp:12-34, 130-144
    nodes, el, _ = M.quad_grid(4, 3)
    q = port.orthogonality(nodes, 2, el)
    assert np.allclose(q["scores"], 90.0, rtol=1e-12) and q["inverted"] == 0
    tri = np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0]], float)
    q = port.orthogonality(tri, 2, M.csr([(M.TRI, [0, 1, 2]), (M.TRI, [0, 2, 3])]))
    assert np.allclose(q["scores"], 90.0, rtol=1e-12)
    deg = np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0], [2, 0.5, 0]], float)
    q = port.orthogonality(deg, 2, M.csr([(M.QUAD, [0, 1, 2, 3]), (M.TRI, [1, 1, 4])]))
    assert q["scores"][1] == 0.0 and q["degenerate"] == 1


def test_orthogonality_invariance(port):  # test_quality.cpp:36-66
    nodes, el = _sheared_quad_grid()
    b = port.orthogonality(nodes, 2, el)
    a, s = 0.7, nodes.copy()
    moved = np.stack([s[:, 0] * math.cos(a) - s[:, 1] * math.sin(a) + 3.0,
                      s[:, 0] * math.sin(a) + s[:, 1] * math.cos(a) - 1.5, 0 * s[:, 0]], 1)
    assert np.allclose(port.orthogonality(moved, 2, el)["scores"], b["scores"], rtol=1e-10)
    sc = port.orthogonality(nodes * 4.0, 2, el)
    assert np.allclose(sc["scores"], b["scores"], rtol=1e-10)
    assert np.allclose(sc["measures"], 16.0 * b["measures"], rtol=1e-12)


def _ortho_cases():
    rng = np.random.default_rng(4)
    nodes, el = _sheared_quad_grid()
    yield "quad", nodes, 2, el
    bn, bel = M.box_grid(3, 3, 2)
    yield "hex", bn + 0.05 * rng.standard_normal(bn.shape), 3, M.csr(bel)
    # tets / prisms / pyramids sharing faces: split each cube of a 2x2x1 grid
    cn, cel = M.box_grid(2, 2, 1)
    mixed = []
    for k, (_, h) in enumerate(cel):
        if k % 3 == 0:  # 5 tets (oracles.cpp:109-120 split)
            for t in ([0, 1, 3, 4], [2, 3, 1, 6], [5, 4, 6, 1], [7, 6, 4, 3], [1, 3, 4, 6]):
                mixed.append((M.TET, [h[i] for i in t]))
        elif k % 3 == 1:  # 2 prisms
            mixed.append((M.PRISM, [h[0], h[1], h[2], h[4], h[5], h[6]]))
            mixed.append((M.PRISM, [h[0], h[2], h[3], h[4], h[6], h[7]]))
        else:
            mixed.append((M.HEX, h))
    yield "mixed", cn + 0.03 * rng.standard_normal(cn.shape), 3, M.csr(mixed)
    pn = np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0], [0.5, 0.5, 1.0], [0.5, 0.5, -1.0]])
    yield "pyramids", pn, 3, M.csr([(M.PYRAMID, [0, 1, 2, 3, 4]), (M.PYRAMID, [3, 2, 1, 0, 5])])
    w = W.cfg1(0.1)
    yield "cfg1", w.nodes, 2, W.elements(w)


@pytest.mark.parametrize("case", [c[0] for c in _ortho_cases()])
def test_port_matches_reference_orthogonality(port, ref, case):
    name, nodes, dim, el = next(c for c in _ortho_cases() if c[0] == case)
    a, b = port.orthogonality(nodes, dim, el), ref.orthogonality(nodes, dim, el)
    assert np.array_equal(bits(a["scores"]), bits(b["scores"]))
    assert np.array_equal(bits(a["measures"]), bits(b["measures"]))
    assert (a["min"], a["mean"], a["inverted"], a["degenerate"]) == \
        (b["min"], b["mean"], b["inverted"], b["degenerate"])


def test_reference_reports_inverted(golden):  # test_pipeline.cpp:216-228
    assert int(golden["inv_count"]) > 0


# ---- CUDA product ------------------------------------------------------------------
@pytest.mark.gpu
def test_gpu_matches_golden_quality(gpu, golden):
    e = (golden["q_kinds"], golden["q_offsets"], golden["q_conn"])
    m, inv = gpu.signed_measures(golden["q_nodes"], e)
    assert np.array_equal(bits(m), bits(golden["q_measures"]))
    assert inv == int(golden["q_inverted"])
    assert gpu.count_inverted(golden["q_nodes"], e) == inv


@pytest.mark.gpu
@pytest.mark.parametrize("seed,n_elem", [(5, 1), (6, 31), (7, 100_003), (8, 1_000_000)])
def test_gpu_random_mixed(gpu, port, seed, n_elem):
    nodes, e = M.random_mixed(np.random.default_rng(seed), 5000, n_elem)
    m, inv = gpu.signed_measures(nodes, e)
    mo, io = port.signed_measures(nodes, 3, e)
    assert np.array_equal(bits(m), bits(mo)) and inv == io


@pytest.mark.gpu
@pytest.mark.parametrize("make", [lambda: W.cfg1(0.25), lambda: W.cfg2(0.2), lambda: W.cfg3(0.05)])
def test_gpu_workload_meshes(gpu, port, make):
    w = make()
    e = W.elements(w)
    m, inv = gpu.signed_measures(w.nodes, e)
    mo, io = port.signed_measures(w.nodes, w.dim, e)
    assert np.array_equal(bits(m), bits(mo)) and inv == io == 0


@pytest.mark.gpu
def test_gpu_empty_and_canonical(gpu):
    nodes = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], float)
    empty = (np.zeros(0, np.int32), np.zeros(1, np.uint64), np.zeros(1, np.uint64))
    m, inv = gpu.signed_measures(nodes, empty)
    assert len(m) == 0 and inv == 0
    m, inv = gpu.signed_measures(nodes, M.csr([(M.TRI, [0, 1, 2]), (M.TRI, [0, 2, 1]),
                                               (M.LINE, [0, 1])]))
    assert list(m) == [0.5, -0.5, 0.0] and inv == 2


@pytest.mark.gpu
def test_gpu_malformed_elements(gpu):  # validate_mesh messages, mesh.cpp:168-185
    nodes = np.zeros((4, 3))
    with pytest.raises(ValueError, match="wrong node count for hexahedron"):
        gpu.signed_measures(nodes, M.csr([(M.TRI, [0, 1, 2]), (M.HEX, [0, 1, 2, 3])]))
    with pytest.raises(ValueError, match="node index 9 out of range"):
        gpu.signed_measures(nodes, M.csr([(M.TET, [0, 1, 2, 9])]))
    with pytest.raises(ValueError, match="unknown element kind"):
        gpu.signed_measures(nodes, M.csr([(9, [0, 1])]))


@pytest.mark.gpu
def test_gpu_deform_reports_inverted(gpu, golden):  # test_pipeline.cpp:216-228
    nodes, el, wall = M.quad_grid(10, 3, 1.0, 0.05)
    disp = M.wall_bump(nodes, wall, 0.5)
    r = gpu.deform(nodes, 2, wall, disp, (), 0.01, 2, 5000, "c2", 0.3, 0.2,
                   precision=capi.EXACT, elements=el)
    assert np.array_equal(r["nodes"], golden["inv_deformed"])
    assert r["inverted_elements"] == int(golden["inv_count"]) > 0
    # without elements the report counts nothing
    r0 = gpu.deform(nodes, 2, wall, disp, (), 0.01, 2, 5000, "c2", 0.3, 0.2,
                    precision=capi.EXACT)
    assert r0["inverted_elements"] == 0


@pytest.mark.gpu
def test_gpu_deform_cfg1_elements(gpu, ref):
    w = W.cfg1(0.2)
    e = W.elements(w)
    r = gpu.deform(w.nodes, 2, w.surface, w.displacement, (), w.tol, w.levels, w.cap, w.kind,
                   w.R, 5.0, precision=capi.EXACT, elements=e)
    rr = ref.deform(w.nodes, 2, w.surface, w.displacement, (), w.tol, w.levels, w.cap, w.kind,
                    w.R, 5.0, elements=e)
    assert np.array_equal(r["nodes"], rr["nodes"])
    assert r["inverted_elements"] == rr["inverted_elements"]


@pytest.mark.gpu
def test_python_mirror_quality(golden):
    from paper_2107_13887_b200 import icemorph as im

    nodes, el, wall = M.quad_grid(10, 3, 1.0, 0.05)
    mesh = im.Mesh(2, nodes, {"wall": wall}, el)
    assert mesh.num_elements == 30
    assert im.count_inverted(mesh) == 0
    assert all(v > 0 for v in im.signed_measures(mesh))
    f = im.DisplacementField("wall")
    for n, d in zip(wall, M.wall_bump(nodes, wall, 0.5)):
        f.set(n, *d)
    cfg = im.DeformationConfig()
    cfg.tolerance, cfg.levels, cfg.support_radius, cfg.volume_k = 0.01, 2, 0.3, 0.2
    out, rep = im.deform(mesh, f, cfg)
    assert rep.inverted_elements == int(golden["inv_count"])
    assert im.count_inverted(out) == rep.inverted_elements


# ---- orthogonality on the device (quality.cpp:150-236) -----------------------------
ORTHO_TOL = 1e-11  # degrees: CUDA atan2 (<= 2 ulp) vs glibc; everything else exact


@pytest.mark.gpu
@pytest.mark.parametrize("case", [c[0] for c in _ortho_cases()])
def test_gpu_orthogonality_matches_oracle(gpu, port, case):
    name, nodes, dim, el = next(c for c in _ortho_cases() if c[0] == case)
    g, o = gpu.orthogonality(nodes, el), port.orthogonality(nodes, dim, el)
    assert np.abs(g["scores"] - o["scores"]).max() <= ORTHO_TOL
    assert np.array_equal(bits(g["measures"]), bits(o["measures"]))
    assert (g["inverted"], g["degenerate"]) == (o["inverted"], o["degenerate"])
    assert abs(g["min"] - o["min"]) <= ORTHO_TOL and abs(g["mean"] - o["mean"]) <= ORTHO_TOL


@pytest.mark.gpu
def test_gpu_orthogonality_kats(gpu):  # test_quality.cpp:12-34, 130-144
    nodes, el, _ = M.quad_grid(4, 3)
    q = gpu.orthogonality(nodes, el)
    assert np.allclose(q["scores"], 90.0, rtol=1e-12) and q["min"] == pytest.approx(90.0)
    deg = np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0], [2, 0.5, 0]], float)
    q = gpu.orthogonality(deg, M.csr([(M.QUAD, [0, 1, 2, 3]), (M.TRI, [1, 1, 4])]))
    assert q["scores"][1] == 0.0 and q["degenerate"] == 1
    empty = (np.zeros(0, np.int32), np.zeros(1, np.uint64), np.zeros(1, np.uint64))
    q = gpu.orthogonality(deg, empty)
    assert q["min"] == 90.0 and q["mean"] == 90.0 and len(q["scores"]) == 0


@pytest.mark.gpu
def test_gpu_orthogonality_full_size(gpu):
    """cfg2's 1M-node O-mesh (999k quads) and a 3-D wing block: a structured
    undeformed mesh has no degenerate or inverted cells and scores in
    (0, 90]; the mean equals the host sum of the per-element scores."""
    for w in (W.cfg2(), W.cfg3(0.15)):
        e = W.elements(w)
        q = gpu.orthogonality(w.nodes, e)
        s = q["scores"]
        assert q["inverted"] == 0 and q["degenerate"] == 0
        assert (s > 0).all() and (s <= 90.0 + 1e-12).all()
        assert q["mean"] == math.fsum(s) / len(s) or abs(q["mean"] - s.mean()) < 1e-9


@pytest.mark.gpu
def test_gpu_deform_quality_reports(gpu, ref):
    """deform with compute_quality: quality_before / quality_after of the
    reference's pipeline (pipeline.cpp:55, 102), exact deformation."""
    nodes, el, wall = M.quad_grid(10, 3, 1.0, 0.05)
    disp = M.wall_bump(nodes, wall, 0.5)
    r = gpu.deform(nodes, 2, wall, disp, (), 0.01, 2, 5000, "c2", 0.3, 0.2,
                   precision=capi.EXACT, elements=el, compute_quality=True)
    before, after = r["quality"]
    qb = ref.orthogonality(nodes, 2, el)
    qa = ref.orthogonality(r["nodes"], 2, el)
    for got, want in ((before, qb), (after, qa)):
        assert abs(got["min"] - want["min"]) <= ORTHO_TOL
        assert abs(got["mean"] - want["mean"]) <= ORTHO_TOL
        assert (got["inverted"], got["degenerate"]) == (want["inverted"], want["degenerate"])
    assert r["inverted_elements"] == qa["inverted"] > 0
