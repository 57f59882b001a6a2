"""``import icemorph`` -- the reference module's name list over the B200
library -- exercised the way the reference's own smoke tests use it
(proj/tests/python/test_smoke.py): generated meshes and displacement fields,
deform + report + convergence CSV, SU2 / VTK / displacement files, quality,
fixed markers, errors."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def im():
    import icemorph

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


def test_generated_deform_report_and_csv(im, tmp_path):  # test_smoke.py:27-52
    mesh = im.gen_airfoil_mesh(1.0, 128, 12)
    assert mesh.num_nodes == 128 * 13
    assert mesh.marker_names() == ["airfoil", "farfield"]
    field = im.gen_sinusoidal_displacement(mesh, "airfoil")
    assert field.max_magnitude() == pytest.approx(0.01, rel=1e-6)
    cfg = im.DeformationConfig()
    cfg.support_radius, cfg.tolerance, cfg.levels, cfg.volume_k = 2.0, 0.1, 3, 5.0
    deformed, report = im.deform(mesh, field, cfg)
    assert report.surface_max_error < 1e-3 and report.inverted_elements == 0
    assert len(report.levels) == 3 and all(l.achieved_error < 0.1 for l in report.levels)
    path = tmp_path / "conv.csv"
    im.write_convergence_csv(report, str(path))
    rows = path.read_text().splitlines()
    assert rows[0] == "level,points,error,seconds"
    assert len(rows) - 1 == report.total_control_points
    im.write_summary(report, str(tmp_path / "summary.txt"))
    assert "total_control_points: %d" % report.total_control_points in (
        tmp_path / "summary.txt").read_text()


def test_generated_files_roundtrip(im, tmp_path):  # test_smoke.py:55-77
    mesh = im.gen_airfoil_mesh(1.0, 64, 8)
    im.write_su2(mesh, str(tmp_path / "m.su2"))
    back = im.read_su2(str(tmp_path / "m.su2"))
    assert back.num_nodes == mesh.num_nodes and back.nodes() == mesh.nodes()
    im.write_vtk(mesh, str(tmp_path / "m.vtk"))
    assert "UNSTRUCTURED_GRID" in (tmp_path / "m.vtk").read_text()
    f = im.DisplacementField("airfoil")
    f.set(3, 0.01, -0.002)
    im.write_displacements(f, mesh.dim, str(tmp_path / "d.txt"))
    g = im.read_displacements(str(tmp_path / "d.txt"), mesh, "airfoil")
    assert tuple(g.entries()[3]) == (0.01, -0.002, 0.0)


def test_generated_quality_and_pinning(im):  # test_smoke.py:80-104
    mesh = im.gen_airfoil_mesh(1.0, 64, 8)
    q = im.orthogonality(mesh)
    assert 0.0 <= q.min_orthogonality_deg <= 90.0 and q.inverted_count == 0
    assert all(m > 0 for m in im.signed_measures(mesh))
    field = im.gen_ice_bump(mesh, "airfoil", height=0.03)
    cfg = im.DeformationConfig()
    cfg.support_radius, cfg.levels, cfg.fixed_markers = 2.0, 2, ["farfield"]
    deformed, _ = im.deform(mesh, field, cfg)
    before, after = mesh.nodes(), deformed.nodes()
    assert all(before[i] == after[i] for i in mesh.marker_nodes("farfield"))
    with pytest.raises(Exception):
        im.gen_sinusoidal_displacement(mesh, "nope")
    with pytest.raises(Exception):
        im.read_su2("does_not_exist.su2")
