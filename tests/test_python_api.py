"""The Python mirror of the reference's icemorph module
(paper_2107_13887_b200/icemorph.py), exercised like the reference's own
smoke tests (proj/tests/python/test_smoke.py) on the hot-path surface."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def im():
    from paper_2107_13887_b200 import icemorph

    return icemorph


def ring_mesh(im, n=128, layers=12):
    nodes, wall, far = [], [], []
    for layer in range(layers + 1):
        r = 1.0 + 0.5 * layer
        for j in range(n):
            t = 2 * math.pi * j / n
            nodes.append((r * math.cos(t), r * math.sin(t), 0.0))
            if layer == 0:
                wall.append(len(nodes) - 1)
            if layer == layers:
                far.append(len(nodes) - 1)
    return im.Mesh(2, nodes, {"airfoil": wall, "farfield": far})


def test_kernel_values(im):  # test_smoke.py:9-15
    assert im.eval_basis("c2", 2.0, 1.0) == 0.1875
    assert im.eval_basis("c0", 1.0, 0.5) == 0.25
    assert im.eval_basis("c2", 1.0, 1.5) == 0.0
    for kind in ("c0", "c2", "c4", "c6"):
        assert im.eval_basis(kind, 1.0, 0.0) == 1.0
        assert im.eval_basis(kind, 1.0, 1.0) == 0.0
    with pytest.raises(ValueError):
        im.eval_basis("c3", 1.0, 0.5)


def test_solve_and_eval_roundtrip(im):  # test_smoke.py:18-24
    points = [(0.0, 0.0, 0.0), (1.0, 0.0, 0.0), (0.3, 0.6, 0.0)]
    disp = [(0.1, 0.0, 0.0), (0.0, -0.2, 0.0), (0.05, 0.05, 0.0)]
    alpha = im.solve_weights(points, disp, "c2", 2.0)
    for p, d in zip(points, disp):
        f = im.eval_interpolant(points, alpha, "c2", 2.0, p)
        assert max(abs(a - b) for a, b in zip(f, d)) < 1e-10


def test_deform_and_report(im):  # test_smoke.py:27-47 (ring mesh instead of gen_airfoil_mesh)
    mesh = ring_mesh(im)
    field = im.DisplacementField("airfoil")
    for n in mesh.marker_nodes("airfoil"):
        x, y, _ = mesh.node(n)
        field.set(n, 0.0, 0.01 * math.sin(15 * math.pi * (x + 1) / 2))
    assert field.max_magnitude() == pytest.approx(0.01, rel=1e-2)
    config = im.DeformationConfig()
    config.support_radius = 2.0
    config.tolerance = 0.1
    config.levels = 3
    config.volume_k = 5.0
    deformed, report = im.deform(mesh, field, config)
    assert report.surface_max_error < 1e-3
    assert 1 <= len(report.levels) <= 3
    for level in report.levels:
        assert level.achieved_error < 0.1
    assert report.total_control_points == sum(l.points for l in report.levels)
    assert deformed.num_nodes == mesh.num_nodes


def test_fixed_markers_pin_nodes(im):  # test_smoke.py:75-88
    mesh = ring_mesh(im, 64, 8)
    field = im.DisplacementField("airfoil")
    for n in mesh.marker_nodes("airfoil"):
        field.set(n, 0.0, 0.03 * math.exp(-((mesh.node(n)[0] + 1.0) ** 2) / 0.01))
    config = im.DeformationConfig()
    config.support_radius = 2.0
    config.levels = 2
    config.fixed_markers = ["farfield"]
    deformed, _ = im.deform(mesh, field, config)
    for i in mesh.marker_nodes("farfield"):
        assert deformed.node(i) == mesh.node(i)


def test_errors_surface(im):  # test_smoke.py:91-105
    mesh = ring_mesh(im, 32, 8)
    with pytest.raises(ValueError):
        im.deform(mesh, im.DisplacementField("nope"), im.DeformationConfig())
    from paper_2107_13887_b200.capi import SolveError

    with pytest.raises(RuntimeError) as e:
        im.solve_weights([(0, 0, 0), (1e-18, 0, 0)], [(1, 0, 0), (2, 0, 0)], "c2", 1.0)
    assert isinstance(e.value, SolveError) and "points 0 and 1" in str(e.value)
