"""The tiled exact volume update (k_volume_exact_tiled) and the resident
volume plan, bit for bit against the reference (wall_distance.cpp:46-64,
rbf.cpp:195-203).

The tiled kernel reorders points spatially, culls tiles / control groups
farther than R and replaces the branches of sqrt / division / the eta >= 1
cut by range-guarded branch-free forms; every case here must still equal the
reference exactly (np.array_equal on the values)."""
import math
import os

import numpy as np
import pytest

from paper_2107_13887_b200 import capi, workloads as W

pytestmark = pytest.mark.gpu


def ref_update(oracle, nodes, d, ctrl, alpha, D, R, psi=0):
    return oracle.update_volume(nodes, d, ctrl, alpha, D, psi, "c2", R)


@pytest.fixture(params=["auto", "gather_tile", "gather_n4", "gather_t64", "no_gather"])
def launch_shape(request, monkeypatch):
    """Every exact kernel: gathered (R < 15 % of the control spread; the
    barrier-free default, its 4-controls-per-stage shape and the tile-streaming
    variant) and group-culled (IMB_NO_GATHER)."""
    if request.param == "no_gather":
        monkeypatch.setenv("IMB_NO_GATHER", "1")
    elif request.param == "gather_tile":
        monkeypatch.setenv("IMB_GATHER", "tile")
    elif request.param == "gather_n4":
        monkeypatch.setenv("IMB_GATHER", "n4")
    elif request.param == "gather_t64":
        monkeypatch.setenv("IMB_GATHER", "t64")
    return request.param


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("R", [0.05, 0.3, 2.0])
def test_random_clouds(gpu, oracle, dim, R, launch_shape):
    rng = np.random.default_rng(int(R * 100) + dim)
    n, nc = 30000, 1500  # several tiles, insertion order not spatial
    nodes = rng.random((n, 3))
    ctrl = rng.random((nc, 3))
    if dim == 2:
        nodes[:, 2] = 0.0
        ctrl[:, 2] = 0.0
    alpha = rng.standard_normal((nc, 3))
    if dim == 2:
        alpha[:, 2] = 0.0
    d = rng.random(n)  # any distances: psi only scales
    i0, v0 = ref_update(oracle, nodes, d, ctrl, alpha, 0.8, R)
    i1, v1 = gpu.update_volume(nodes, d, ctrl, alpha, 0.8, 0, "c2", R, capi.EXACT)
    assert np.array_equal(i0, i1) and np.array_equal(v0, v1)


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("m,scale", [(-2, 1.0), (0, 1.0), (3, 1.0), (-64, 2.0 ** -62), (64, 2.0 ** 63),
                                     (10, 2.0 ** -300), (-3, 1e-9), (60, 2.0 ** -520), (64, 2.0 ** -440)])
def test_power_of_two_radius(gpu, oracle, dim, m, scale, launch_shape, monkeypatch):
    """R = 2^m: the exact kernels pre-scale points and tiles by 1/R and drop
    the division (volume.cu ScaleTile); eta must not change by a bit, also when
    the scaled coordinates leave the normal range's comfortable middle
    (clouds of extent `scale`, so in-support pairs exist only when scale ~ R)."""
    rng = np.random.default_rng(97 + m + dim)
    n, nc = 20000, 700
    nodes = rng.random((n, 3)) * scale
    ctrl = rng.random((nc, 3)) * scale
    if dim == 2:
        nodes[:, 2] = 0.0
        ctrl[:, 2] = 0.0
    alpha = rng.standard_normal((nc, 3))
    if dim == 2:
        alpha[:, 2] = 0.0
    d = rng.random(n)
    R = 2.0 ** m
    i0, v0 = ref_update(oracle, nodes, d, ctrl, alpha, 0.8, R)
    i1, v1 = gpu.update_volume(nodes, d, ctrl, alpha, 0.8, 0, "c2", R, capi.EXACT)
    assert np.array_equal(i0, i1) and np.array_equal(v0, v1)
    monkeypatch.setenv("IMB_NO_PRESCALE", "1")
    i2, v2 = gpu.update_volume(nodes, d, ctrl, alpha, 0.8, 0, "c2", R, capi.EXACT)
    assert np.array_equal(i0, i2) and np.array_equal(v0, v2)


@pytest.mark.parametrize("R", [40.0, 10.0, 2.5, 1.75, 3.0])
def test_two_operation_division(gpu, oracle, R, monkeypatch):
    """Global support with a radius whose significand is a multiple of 4: the
    3-D kernel forms eta = d / R with exact::div2 (two operations, proven
    correctly rounded for such divisors, tests/test_div2.py); it must equal
    the reference and the three-operation form bit for bit."""
    rng = np.random.default_rng(int(R * 4))
    n, nc = 40000, 900
    nodes = rng.random((n, 3)) * [1.0, 1.5, 0.3]
    ctrl = rng.random((nc, 3)) * [1.0, 1.5, 0.3]
    alpha = rng.standard_normal((nc, 3))
    d = rng.random(n)
    i0, v0 = ref_update(oracle, nodes, d, ctrl, alpha, 0.8, R)
    i1, v1 = gpu.update_volume(nodes, d, ctrl, alpha, 0.8, 0, "c2", R, capi.EXACT)
    assert np.array_equal(i0, i1) and np.array_equal(v0, v1)
    monkeypatch.setenv("IMB_NO_DIV2", "1")
    i2, v2 = gpu.update_volume(nodes, d, ctrl, alpha, 0.8, 0, "c2", R, capi.EXACT)
    assert np.array_equal(i0, i2) and np.array_equal(v0, v2)


def test_boundary_pairs(gpu, oracle, launch_shape):
    """eta exactly 1, just below / above 1, coincident points (s = 0), tiny
    distances (s below the 2^-900 clamp), negative zero coordinates."""
    R = 0.5
    ctrl = np.array([[0.0, 0.0, 0.0], [1.0, 1.0, 1.0]])
    alpha = np.array([[1.0, -2.0, 3.0], [0.25, 0.5, -0.75]])
    ulp = np.nextafter(0.5, 1.0) - 0.5
    pts = [[0.0, 0.0, 0.0], [0.5, 0.0, 0.0], [0.0, 0.5, 0.0], [0.0, 0.0, 0.5],
           [0.5 - ulp, 0.0, 0.0], [0.5 + ulp, 0.0, 0.0], [1e-160, 0.0, 0.0],
           [-0.0, -0.0, -0.0], [1.0, 1.0, 1.0], [1.0, 1.0, 1.0 - 1e-170], [1.5, 1.0, 1.0],
           [0.3, 0.4, 0.0], [0.25, 0.25, 0.25]]
    nodes = np.array(pts, float)
    d = np.zeros(len(nodes))
    i0, v0 = ref_update(oracle, nodes, d, ctrl, alpha, 1.0, R)
    i1, v1 = gpu.update_volume(nodes, d, ctrl, alpha, 1.0, 0, "c2", R, capi.EXACT)
    assert np.array_equal(i0, i1) and np.array_equal(v0, v1)
    assert (v1[1] == 0).all() and (v1[0] == alpha[0]).all()  # eta = 1 -> phi = +0


@pytest.mark.parametrize("kind", ["c0", "c4", "c6"])
def test_other_kinds(gpu, oracle, kind):
    rng = np.random.default_rng(3)
    nodes, ctrl = rng.random((8000, 3)), rng.random((700, 3))
    alpha = rng.standard_normal((700, 3))
    d = np.zeros(len(nodes))
    i0, v0 = oracle.update_volume(nodes, d, ctrl, alpha, 1.0, 0, kind, 0.25)
    i1, v1 = gpu.update_volume(nodes, d, ctrl, alpha, 1.0, 0, kind, 0.25, capi.EXACT)
    assert np.array_equal(i0, i1) and np.array_equal(v0, v1)


def test_cfg1_levels_golden(gpu, golden):
    """The reference's own cfg1 (30 %) control sets, real airfoil geometry."""
    g = golden
    nodes, surf = g["cfg1s_nodes"], g["cfg1s_surface"]
    d = gpu.build_distance_index(nodes, 2, surf)
    pos = nodes[surf]
    for l in range(int(g["cfg1s_nlevels"])):
        c, a = pos[g[f"cfg1s_l{l}_idx"]], g[f"cfg1s_l{l}_alpha"]
        i1, v1 = gpu.update_volume(nodes, d, c, a, 1.0, 0, "c2", 0.5, capi.EXACT)
        i2, v2 = gpu.update_volume(nodes, d, c, a, 1.0, 0, "c2", 0.5, capi.EXACT)
        assert np.array_equal(v1, v2) and np.array_equal(i1, np.flatnonzero(d < 1.0))


def test_cfg1_levels_reference(gpu, oracle, golden, launch_shape):
    g = golden
    nodes, surf = g["cfg1s_nodes"], g["cfg1s_surface"]
    d = gpu.build_distance_index(nodes, 2, surf)
    pos = nodes[surf]
    for l in range(int(g["cfg1s_nlevels"])):
        c, a = pos[g[f"cfg1s_l{l}_idx"]], g[f"cfg1s_l{l}_alpha"]
        i0, v0 = oracle.update_volume(nodes, d, c, a, 1.0, 1, "c2", 0.5)
        i1, v1 = gpu.update_volume(nodes, d, c, a, 1.0, 1, "c2", 0.5, capi.EXACT)
        assert np.array_equal(i0, i1) and np.array_equal(v0, v1)


@pytest.mark.parametrize("precision", [capi.EXACT, capi.FP64])
def test_volume_plan_levels(gpu, oracle, golden, precision, launch_shape):
    """The resident plan (bench.py's timed path): one step over two levels
    accumulates ((0 + dV_0) + dV_1) per node, dV_l from the reference."""
    g = golden
    nodes, surf = g["cfg1s_nodes"], g["cfg1s_surface"]
    D = 1.0
    plan = capi.VolumePlan(gpu, nodes, 2, surf, cutoff=D)
    d = plan.distances()
    assert np.array_equal(d < D, gpu.build_distance_index(nodes, 2, surf) < D)
    pos = nodes[surf]
    expect = np.zeros((len(nodes), 3))
    levels = range(int(g["cfg1s_nlevels"]))
    for l in levels:
        c, a = pos[g[f"cfg1s_l{l}_idx"]], g[f"cfg1s_l{l}_alpha"]
        plan.set_level(l, c, a, D, 0, "c2", 0.5, precision)
        i0, v0 = oracle.update_volume(nodes, d, c, a, D, 0, "c2", 0.5)
        expect[i0] = expect[i0] + v0
    plan.reset_field()
    st = plan.run_steps(1, "c2", 0.5, precision, flush_l2=False)
    assert st["active"][0] == int((d < D).sum())
    got = plan.field()
    if precision == capi.EXACT:
        assert np.array_equal(got, expect)
    else:
        assert np.abs(got - expect).max() <= 1e-10 * np.abs(expect).max()
    # the flop-roofline pair count does not depend on the tile format
    assert plan.count_support(0, "c2", 0.5)[0] > 0


def test_volume_plan_single_level_run(gpu, oracle):
    rng = np.random.default_rng(9)
    nodes = rng.random((20000, 3))
    surf = np.arange(0, 20000, 50)
    plan = capi.VolumePlan(gpu, nodes, 3, surf, cutoff=math.inf)
    d = plan.distances()
    ctrl, alpha = nodes[surf[:200]], rng.standard_normal((200, 3))
    plan.set_controls(ctrl, alpha)
    i0, v0 = oracle.update_volume(nodes, d, ctrl, alpha, 0.3, 0, "c2", 0.2)
    for prec in (capi.EXACT, capi.FP64):
        plan.reset_field()
        na, _ = plan.run(0.3, 0, "c2", 0.2, prec)
        assert na == len(i0)
        f = plan.field()[i0]
        if prec == capi.EXACT:
            assert np.array_equal(f, v0)
        else:
            assert np.abs(f - v0).max() <= 1e-10 * np.abs(v0).max()


def test_cfg2_levels_slice_matches_reference(gpu, oracle):
    """Full BASELINE cfg2 geometry and the device greedy's own levels 0-1
    (166 / 1425 controls; bit-identical to the reference's selection,
    test_cfg2_full_selection): the exact volume update on 40k mesh nodes
    closest to the wall equals the reference's update_volume bit for bit."""
    w = W.cfg2()
    pos = w.nodes[w.surface]
    m = gpu.run_multilevel(pos, w.displacement, w.tol, 2, w.cap, w.kind, w.R)
    d = gpu.build_distance_index(w.nodes, 2, w.surface)
    pick = np.sort(np.argsort(d)[:40000])
    nodes, dd = np.ascontiguousarray(w.nodes[pick]), np.ascontiguousarray(d[pick])
    for lv in m.levels:
        c = pos[lv.control_indices]
        i0, v0 = oracle.update_volume(nodes, dd, c, lv.alpha, w.D, w.psi_kind, "c2", w.R,
                                      nthreads=os.cpu_count() or 1)
        i1, v1 = gpu.update_volume(nodes, dd, c, lv.alpha, w.D, w.psi_kind, "c2", w.R, capi.EXACT)
        assert np.array_equal(i0, i1) and np.array_equal(v0, v1)


def test_update_volume_pinned_buffers(gpu):
    """Page-locked inputs / outputs take the direct-DMA path of the host
    transfers (host_io.cu); results equal the staged (pageable) path."""
    import torch

    rng = np.random.default_rng(12)
    nodes, ctrl = rng.random((50000, 3)), rng.random((900, 3))
    alpha, d = rng.standard_normal((900, 3)), rng.random(50000)
    i0, v0 = gpu.update_volume(nodes, d, ctrl, alpha, 0.7, 0, "c2", 0.2, capi.EXACT)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
    out = (torch.empty(50000, dtype=torch.int64, pin_memory=True).numpy().view(np.uint64),
           torch.empty((50000, 3), dtype=torch.float64, pin_memory=True).numpy())
    i1, v1 = gpu.update_volume(pin(nodes), pin(d), ctrl, alpha, 0.7, 0, "c2", 0.2, capi.EXACT, out=out)
    assert np.array_equal(i0, i1) and np.array_equal(v0, v1)
    planar = nodes.copy()
    planar[:, 2] = 0.0
    c2, a2 = ctrl.copy(), alpha.copy()
    c2[:, 2] = a2[:, 2] = 0.0
    i2, v2 = gpu.update_volume(planar, d, c2, a2, 0.7, 0, "c2", 0.2, capi.FP64)
    i3, v3 = gpu.update_volume(pin(planar), pin(d), c2, a2, 0.7, 0, "c2", 0.2, capi.FP64, out=out)
    assert np.array_equal(i2, i3) and np.array_equal(v2, v3)  # planar detection on the direct path
