"""Pin the oracle before trusting it: the plain-C restatement (and the
reference build) against the known-answer values of the reference's own
tests (proj/tests/*.cpp) and against the golden fixtures generated from the
reference (tests/golden/make_golden.py)."""
import math

import numpy as np
import pytest

FLAVOURS = ["port", "ref"]


@pytest.fixture(params=FLAVOURS)
def orc(request):
    return request.getfixturevalue(request.param)


# ---- rbf KATs: test_rbf.cpp ---------------------------------------------------
def test_wendland_values(orc):  # test_rbf.cpp:40-52
    assert orc.eval_wendland("c2", 0.0) == 1.0
    assert orc.eval_wendland("c2", 0.5) == 0.1875
    assert orc.eval_wendland("c0", 0.5) == 0.25
    assert orc.eval_wendland("c2", 1.2) == 0.0
    for k in ("c0", "c2", "c4", "c6"):
        assert orc.eval_wendland(k, 0.0) == 1.0
        assert orc.eval_wendland(k, 1.0) == 0.0
        assert orc.eval_wendland(k, 1.0 + 1e-12) == 0.0
        assert orc.eval_wendland(k, 37.5) == 0.0


def test_wendland_monotone(orc):  # test_rbf.cpp:54-65
    for k in ("c0", "c2", "c4", "c6"):
        prev = orc.eval_wendland(k, 0.0)
        for i in range(1, 1001):
            v = orc.eval_wendland(k, i / 1000.0)
            assert v <= prev + 1e-15
            prev = v


def test_two_point_solve(orc):  # test_rbf.cpp:96-119
    pts = [[0, 0, 0], [1, 0, 0]]
    a = orc.solve_weights(pts, [[1, 0, 0], [0, 0, 0]], "c2", 2.0)
    b = 0.1875
    assert a[0, 0] == pytest.approx(1 / (1 - b * b), rel=1e-12)
    assert a[1, 0] == pytest.approx(-b / (1 - b * b), rel=1e-12)
    assert a[0, 0] == pytest.approx(1.036437, rel=1e-6)
    assert a[1, 0] == pytest.approx(-0.194332, rel=1e-5)
    assert a[0, 1] == 0.0
    mid = orc.eval_interpolant(pts, a, "c2", 2.0, [[0.5, 0, 0]])
    assert mid[0, 0] == pytest.approx(0.6328125 / 1.1875, rel=1e-12)
    assert mid[0, 0] == pytest.approx(0.532895, rel=1e-6)


def test_zero_displacement_short_circuit(orc):  # test_rbf.cpp:121-127
    a = orc.solve_weights([[0, 0, 0], [0.25, 0, 0], [0.5, 0, 0]], np.zeros((3, 3)), "c2", 1.0)
    assert (a == 0).all()


def test_duplicate_points_error(orc):  # test_rbf.cpp:223-229
    with pytest.raises(Exception) as e:
        orc.solve_weights([[0, 0, 0], [1e-18, 0, 0]], [[1, 0, 0], [2, 0, 0]], "c2", 1.0)
    assert "points 0 and 1" in str(e.value)


def test_isolated_controls_exact(orc):  # test_rbf.cpp:165-175
    pts = [[0, 0, 0], [10, 0, 0]]
    a = orc.solve_weights(pts, [[0.5, -0.25, 0], [1, 2, 0]], "c2", 2.0)
    q = orc.eval_interpolant(pts, a, "c2", 2.0, [[0, 0, 0], [10, 0, 0], [5, 0, 0], [0, 100, 0]])
    assert (q[0] == a[0]).all() and (q[1] == a[1]).all()
    assert (q[2] == 0).all() and (q[3] == 0).all()


# ---- greedy KATs: test_greedy.cpp ---------------------------------------------
def test_three_collinear(orc):  # test_greedy.cpp:38-51
    g = orc.greedy_level([[0, 0, 0], [0.5, 0, 0], [1, 0, 0]], [[0, 0, 0], [0, 1, 0], [0, 0, 0]],
                         0.1, 5000, "c2", 2.0)
    assert list(g.control_indices[:2]) == [0, 1]
    assert g.achieved_error < 0.1


def test_zero_target(orc):  # test_greedy.cpp:83-93
    g = orc.greedy_level([[0, 0, 0], [1, 0, 0], [2, 0, 0]], np.zeros((3, 3)), 0.1, 5000, "c2", 2.0)
    assert list(g.control_indices) == [0]
    assert g.achieved_error == 0.0 and not g.cap_hit
    assert (g.alpha == 0).all() and len(g.record_error) == 1


def test_cap_recorded(orc):  # test_greedy.cpp:104-112
    t = 2 * np.pi * np.arange(40) / 40
    pos = np.stack([np.cos(t), np.sin(t), 0 * t], 1)
    tgt = np.stack([0 * t, 0.1 * np.sin(2 * t) + 0.05 * np.cos(t), 0 * t], 1)
    g = orc.greedy_level(pos, tgt, 1e-6, 3, "c2", 4.0)
    assert len(g.control_indices) == 3 and g.cap_hit


def test_duplicate_surface_points(orc):  # test_greedy.cpp:123-129
    with pytest.raises(Exception) as e:
        orc.greedy_level([[0, 0, 0], [0, 0, 0], [1, 0, 0]], [[0, 1, 0], [0, 2, 0], [0, 0, 0]],
                         1e-9, 5000, "c2", 2.0)
    assert "too close" in str(e.value)


def test_multilevel_telescopes(orc):  # test_greedy.cpp:131-150
    t = 2 * np.pi * np.arange(80) / 80
    pos = np.stack([np.cos(t), np.sin(t), 0 * t], 1)
    tgt = np.stack([0 * t, 0.1 * np.sin(2 * t) + 0.05 * np.cos(t), 0 * t], 1)
    m = orc.run_multilevel(pos, tgt, 0.3, 3, 5000, "c2", 3.0)
    assert m.levels and all(l.achieved_error < 0.3 and not l.cap_hit for l in m.levels)
    resmax = np.linalg.norm(m.final_residual, axis=1).max()
    assert resmax < 0.3 ** len(m.levels) * m.target_max


# ---- wall distance KATs: test_wall_distance.cpp ---------------------------------
def test_hand_wall_distance(orc):  # test_wall_distance.cpp:29-39
    d = orc.build_distance_index([[0, 0, 0], [1, 0, 0], [0.5, 1, 0], [4, 0, 0]], 2, [0, 1])
    assert d[0] == 0.0 and d[1] == 0.0
    assert d[2] == pytest.approx(math.sqrt(1.25), rel=1e-15)
    assert d[3] == 3.0


def test_update_volume_kats(orc):  # test_wall_distance.cpp:62-115
    nodes = [[0, 0, 0], [0, 0.05, 0], [0, 0.2, 0], [0, 5, 0]]
    d = orc.build_distance_index(nodes, 2, [0])
    idx, val = orc.update_volume(nodes, d, [[0, 0, 0]], [[0, 0.7, 0]], 0.1, 0, "c2", 2.0)
    assert list(idx) == [0, 1]
    assert (val[0] == [0, 0.7, 0]).all()
    assert val[1, 1] == pytest.approx(0.5 * 0.7 * orc.eval_wendland("c2", 0.025), rel=1e-14)
    nodes = [[0, 0, 0], [0, 0.5, 0]]
    d = orc.build_distance_index(nodes, 2, [0])
    idx, val = orc.update_volume(nodes, d, [[0, 1.5, 0]], [[0.3, 0, 0]], 1.0, 0, "c2", 2.0)
    assert val[list(idx).index(1), 0] == pytest.approx(0.5 * 0.3 * 0.1875, rel=1e-14)
    idx, val = orc.update_volume(nodes, d, [[0, 0, 0]], [[0, 0, 0]], 0.0, 0, "c2", 1.0)
    assert len(idx) == 0


# ---- golden fixtures from the reference -----------------------------------------
def test_port_matches_golden(port, golden):
    g = golden
    for t in range(4):
        r = port.greedy_level(g[f"greedy{t}_pos"], g[f"greedy{t}_tgt"], 0.05, 5000, "c2", 1.5)
        assert np.array_equal(r.control_indices, g[f"greedy{t}_idx"])
        assert np.array_equal(r.alpha, g[f"greedy{t}_alpha"])
        assert np.array_equal(r.record_error, g[f"greedy{t}_err"])
        assert np.array_equal(r.residual, g[f"greedy{t}_res"])
    m = port.run_multilevel(g["circle_pos"], g["circle_tgt"], 0.3, 3, 5000, "c2", 3.0)
    assert len(m.levels) == int(g["circle_nlevels"])
    for l, lv in enumerate(m.levels):
        assert np.array_equal(lv.control_indices, g[f"circle_l{l}_idx"])
        assert np.array_equal(lv.alpha, g[f"circle_l{l}_alpha"])
    assert np.array_equal(m.final_residual, g["circle_final"])
    assert np.array_equal(port.solve_weights(g["sw_pts"], g["sw_disp"], "c2", 0.9), g["sw_alpha"])
    d = port.build_distance_index(g["wd_nodes"], 3, np.arange(1000), nthreads=4)
    assert np.array_equal(d, g["wd_dist"])
    for psi in (0, 1):
        i, v = port.update_volume(g["wd_nodes"], g["wd_dist"], g["wd_nodes"][:40], g["uv_alpha"],
                                  0.35, psi, "c2", 0.5, nthreads=3)
        assert np.array_equal(i, g[f"uv{psi}_idx"]) and np.array_equal(v, g[f"uv{psi}_val"])
    surf = g["cfg1s_nodes"][g["cfg1s_surface"]]
    m = port.run_multilevel(surf, g["cfg1s_disp"], 1e-3, 2, 5000, "c2", 0.5)
    assert len(m.levels) == int(g["cfg1s_nlevels"])
    for l, lv in enumerate(m.levels):
        assert np.array_equal(lv.control_indices, g[f"cfg1s_l{l}_idx"])
        assert np.array_equal(lv.alpha, g[f"cfg1s_l{l}_alpha"])


def test_port_matches_reference_random(port, ref):
    rng = np.random.default_rng(99)
    for dim in (2, 3):
        pos = rng.random((120, 3))
        if dim == 2:
            pos[:, 2] = 0
        tgt = rng.standard_normal((120, 3)) * 0.01
        if dim == 2:
            tgt[:, 2] = 0
        a = port.run_multilevel(pos, tgt, 0.02, 3, 5000, "c2", 0.4)
        b = ref.run_multilevel(pos, tgt, 0.02, 3, 5000, "c2", 0.4)
        assert len(a.levels) == len(b.levels)
        for la, lb in zip(a.levels, b.levels):
            assert np.array_equal(la.control_indices, lb.control_indices)
            assert np.array_equal(la.alpha, lb.alpha)
            assert np.array_equal(la.record_error, lb.record_error)
        assert np.array_equal(a.final_residual, b.final_residual)
    for kind in ("c0", "c4", "c6"):
        p = rng.random((25, 3))
        d = rng.standard_normal((25, 3))
        assert np.array_equal(port.solve_weights(p, d, kind, 0.8), ref.solve_weights(p, d, kind, 0.8))


@pytest.mark.parametrize("name", ["cfg3", "cfg4"])
def test_threaded_port_matches_wing_prefix(port, name):
    """The port with a threaded greedy sweep (used to make the full-size wing
    fixture) reproduces the reference's own 300-point / 2-level prefix on the
    full cfg3 / cfg4 surfaces bit for bit (tests/golden/make_wing_selection.py)."""
    import hashlib
    import os

    from paper_2107_13887_b200 import workloads as W

    fx = np.load(os.path.join(os.path.dirname(__file__), "golden", "wing_prefix_reference.npz"))
    pos, disp, R, tol, _ = W.wing_surface_case(name)
    port.set_sweep_threads(max(2, min(8, os.cpu_count() or 2)))
    try:
        m = port.run_multilevel(pos, disp, tol, 2, 300, "c2", R)
    finally:
        port.set_sweep_threads(1)
    assert len(m.levels) == int(fx[f"{name}_nlevels"])
    for l, lv in enumerate(m.levels):
        assert np.array_equal(lv.control_indices, fx[f"{name}_idx{l}"])
        assert np.array_equal(lv.alpha, fx[f"{name}_alpha{l}"])
        assert np.array_equal(lv.record_error, fx[f"{name}_rec{l}"])
    dg = hashlib.sha256(np.ascontiguousarray(m.final_residual).tobytes()).hexdigest()
    assert dg == str(fx[f"{name}_residual_sha"])
