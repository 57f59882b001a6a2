"""The FP32 evaluation mode (IM_FP32, k_volume_f32) against the CPU oracle.

North star: "displacements must agree to a relative 1e-10 in FP64 (1e-5 if an
FP32 evaluation mode is offered)".  FP32 has no reference implementation
(SURVEY §8(c)), so it is held to the FP64 oracle (the unmodified reference,
oracle/_ref, or its plain-C restatement) at 1e-5 relative to max |reference|,
on well-conditioned weights (the raw kernel sweep's alpha ~ N(0,1)); the
active set is bit-exact (it does not depend on the arithmetic mode).
"""
import math

import numpy as np
import pytest

from paper_2107_13887_b200 import capi, workloads as W

pytestmark = pytest.mark.gpu
F32_TOL = 1e-5  # north-star FP32 tolerance, relative to max |reference|


def rel_err(a, b):
    scale = np.abs(b).max() if b.size else 0.0
    return np.abs(a - b).max() / scale if scale > 0 else np.abs(a - b).max()


@pytest.mark.parametrize("R,D", [(0.05, 0.1), (0.2, 0.5), (1.0, math.inf), (math.inf, 0.5),
                                 (0.05, math.inf)])
def test_update_volume_raw_fp32(gpu, oracle, R, D):
    """Raw kernel sweep shapes (BASELINE configs[4], FP32 column) at oracle size."""
    raw = W.raw(700, 40000, R if math.isfinite(R) else 1e300, D, n_wall=800)
    nodes = np.vstack([raw["vol"], raw["wall"]])
    surface = np.arange(len(raw["vol"]), len(nodes))
    d = gpu.build_distance_index(nodes, 3, surface)
    Rv = raw["R"]
    i0, v0 = oracle.update_volume(nodes, d, raw["ctrl"], raw["alpha"], D, 0, "c2", Rv)
    i1, v1 = gpu.update_volume(nodes, d, raw["ctrl"], raw["alpha"], D, 0, "c2", Rv, capi.FP32)
    assert np.array_equal(i0, i1)
    assert rel_err(v1, v0) < F32_TOL


@pytest.mark.parametrize("kind", ["c0", "c2", "c4", "c6"])
@pytest.mark.parametrize("R", [0.05, 0.3, 1.0, 1e6])
def test_eval_interpolant_fp32(gpu, oracle, kind, R):
    rng = np.random.default_rng(7)
    ctrl, alpha = rng.random((600, 3)), rng.standard_normal((600, 3))
    q = rng.random((4000, 3)) * 2 - 0.5
    ref = oracle.eval_interpolant(ctrl, alpha, kind, R, q)
    assert rel_err(gpu.eval_interpolant(ctrl, alpha, kind, R, q, capi.FP32), ref) < F32_TOL


def test_fp32_large_coordinates(gpu, oracle):
    """Coordinates far from the origin: the FP32 differences are formed
    relative to each tile's origin in FP64, so an offset of 1e4 R costs nothing."""
    rng = np.random.default_rng(3)
    off = np.array([1e3, -2e3, 5e2])
    ctrl, alpha = rng.random((500, 3)) + off, rng.standard_normal((500, 3))
    q = rng.random((3000, 3)) * 1.4 - 0.2 + off
    ref = oracle.eval_interpolant(ctrl, alpha, "c2", 0.1, q)
    assert rel_err(gpu.eval_interpolant(ctrl, alpha, "c2", 0.1, q, capi.FP32), ref) < F32_TOL


def test_fp32_edge_cases(gpu, oracle):
    # a query on a control -> phi(0) = 1 (alpha rounded to FP32); a query at
    # exactly R or beyond -> exactly 0; empty control set -> zeros
    c = np.array([[0.0, 0.0, 0.0]])
    a = np.array([[0.3, -0.2, 0.1]])
    q = np.array([[0.0, 0.0, 0.0], [0.5, 0.0, 0.0], [0.25, 0.0, 0.0], [3.0, 0.0, 0.0]])
    out = gpu.eval_interpolant(c, a, "c2", 0.5, q, capi.FP32)
    assert np.array_equal(out[0], a[0].astype(np.float32).astype(np.float64))
    assert (out[1] == 0).all() and (out[3] == 0).all()
    assert rel_err(out, oracle.eval_interpolant(c, a, "c2", 0.5, q)) < F32_TOL
    z = gpu.eval_interpolant(np.zeros((0, 3)), np.zeros((0, 3)), "c2", 1.0, q, capi.FP32)
    assert (z == 0).all()


def test_fp32_planar(gpu, oracle):
    """Planar input takes the 2-D FP32 kernel."""
    rng = np.random.default_rng(11)
    nodes = np.zeros((30000, 3))
    nodes[:, :2] = rng.random((30000, 2)) * 2 - 0.5
    surface = np.arange(29000, 30000)
    d = gpu.build_distance_index(nodes, 2, surface)
    ctrl = np.zeros((400, 3))
    ctrl[:, :2] = rng.random((400, 2))
    alpha = np.zeros((400, 3))
    alpha[:, :2] = rng.standard_normal((400, 2))
    i0, v0 = oracle.update_volume(nodes, d, ctrl, alpha, 0.6, 0, "c2", 0.15)
    i1, v1 = gpu.update_volume(nodes, d, ctrl, alpha, 0.6, 0, "c2", 0.15, capi.FP32)
    assert np.array_equal(i0, i1) and rel_err(v1, v0) < F32_TOL
    assert (v1[:, 2] == 0).all()


def test_fp32_resident_plan(gpu, oracle):
    """bench.py's timed path: two levels accumulated in the resident field."""
    raw = W.raw(1200, 60000, 0.2, 0.5, n_wall=1000)
    nodes = np.vstack([raw["vol"], raw["wall"]])
    surface = np.arange(len(raw["vol"]), len(nodes))
    plan = capi.VolumePlan(gpu, nodes, 3, surface, cutoff=0.5)
    d = plan.distances()
    rng = np.random.default_rng(2)
    levels = [(raw["ctrl"], raw["alpha"]), (rng.random((300, 3)), rng.standard_normal((300, 3)))]
    for l, (c, a) in enumerate(levels):
        plan.set_level(l, c, a, 0.5, 0, "c2", 0.2, capi.FP32)
    plan.reset_field()
    plan.run_steps(1, "c2", 0.2, capi.FP32, flush_l2=False)
    got = plan.field()
    ref = np.zeros_like(nodes)
    for c, a in levels:
        i, v = oracle.update_volume(nodes, d, c, a, 0.5, 0, "c2", 0.2)
        ref[i] += v
    assert rel_err(got, ref) < F32_TOL
    # a level packed for FP32 cannot be run in the exact mode
    with pytest.raises(ValueError, match="different precision"):
        plan.run_steps(1, "c2", 0.2, capi.EXACT, flush_l2=False)
    plan.close()


def test_invalid_precision(gpu):
    c = np.array([[0.0, 0.0, 0.0]])
    with pytest.raises(ValueError, match="unknown precision"):
        gpu.eval_interpolant(c, c, "c2", 1.0, c, 7)
