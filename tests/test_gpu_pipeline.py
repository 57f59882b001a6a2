"""The pipelined im_update_volume (node chunks: uploads, kernels and downloads
overlapped on three streams) against the oracle, forced onto small inputs
with IMB_E2E_CHUNK so every chunking corner is exercised: chunks without
active nodes, planar and non-planar chunks, all three precisions, pageable
and page-locked output buffers.  The entries must equal the reference's
bit for bit in the exact mode (order included: ascending node ids).
"""
import math

import numpy as np
import pytest

from paper_2107_13887_b200 import capi, workloads as W

pytestmark = pytest.mark.gpu


def rel_err(a, b):
    scale = np.abs(b).max() if b.size else 0.0
    return np.abs(a - b).max() / scale if scale > 0 else np.abs(a - b).max()


@pytest.fixture
def chunked(monkeypatch):
    def set_chunk(n):
        monkeypatch.setenv("IMB_E2E_CHUNK", str(n))
    return set_chunk


@pytest.mark.parametrize("chunk", [4096, 7000, 25000])
@pytest.mark.parametrize("R,D", [(0.05, 0.1), (0.3, 0.5), (math.inf, math.inf)])
def test_pipelined_exact_raw(gpu, oracle, chunked, chunk, R, D):
    raw = W.raw(600, 40000, R if math.isfinite(R) else 1e300, D, n_wall=800)
    nodes = np.vstack([raw["vol"], raw["wall"]])
    surface = np.arange(len(raw["vol"]), len(nodes))
    d = gpu.build_distance_index(nodes, 3, surface)
    Rv = raw["R"]
    i0, v0 = oracle.update_volume(nodes, d, raw["ctrl"], raw["alpha"], D, 0, "c2", Rv)
    chunked(chunk)
    i1, v1 = gpu.update_volume(nodes, d, raw["ctrl"], raw["alpha"], D, 0, "c2", Rv, capi.EXACT)
    assert np.array_equal(i0, i1) and np.array_equal(v0, v1)
    i2, v2 = gpu.update_volume(nodes, d, raw["ctrl"], raw["alpha"], D, 0, "c2", Rv, capi.FP64)
    assert np.array_equal(i0, i2) and rel_err(v2, v0) < 1e-10
    i3, v3 = gpu.update_volume(nodes, d, raw["ctrl"], raw["alpha"], D, 0, "c2", Rv, capi.FP32)
    assert np.array_equal(i0, i3) and rel_err(v3, v0) < 1e-5


def test_pipelined_airfoil_levels(gpu, oracle, golden, chunked):
    """cfg1-shaped planar mesh with the reference's own multilevel weights (the
    ill-conditioned case): exact mode bit-identical through the pipeline, with
    chunks far from the wall holding no active node."""
    g = golden
    nodes, surf = g["cfg1s_nodes"], g["cfg1s_surface"]
    d = gpu.build_distance_index(nodes, 2, surf)
    pos = nodes[surf]
    chunked(1000)
    for l in range(int(g["cfg1s_nlevels"])):
        c, a = pos[g[f"cfg1s_l{l}_idx"]], g[f"cfg1s_l{l}_alpha"]
        for D in (0.3, 1.0):
            i0, v0 = oracle.update_volume(nodes, d, c, a, D, 0, "c2", 0.5)
            i1, v1 = gpu.update_volume(nodes, d, c, a, D, 0, "c2", 0.5, capi.EXACT)
            assert np.array_equal(i0, i1) and np.array_equal(v0, v1)


def test_pipelined_mixed_planar_chunks(gpu, oracle, chunked):
    """Half the mesh planar, half not: chunks take the 2-D or 3-D kernels."""
    rng = np.random.default_rng(4)
    nodes = rng.random((30000, 3)) * 2 - 0.5
    nodes[:15000, 2] = 0.0
    surface = np.arange(29000, 30000)
    d = gpu.build_distance_index(nodes, 3, surface)
    ctrl = rng.random((300, 3))
    ctrl[:, 2] = 0.0
    alpha = rng.standard_normal((300, 3))
    alpha[:, 2] = 0.0
    i0, v0 = oracle.update_volume(nodes, d, ctrl, alpha, 0.8, 1, "c2", 0.25)
    chunked(5000)
    i1, v1 = gpu.update_volume(nodes, d, ctrl, alpha, 0.8, 1, "c2", 0.25, capi.EXACT)
    assert np.array_equal(i0, i1) and np.array_equal(v0, v1)


def test_pipelined_pinned_buffers(gpu, oracle, chunked):
    """Page-locked inputs and outputs (the bench's e2e arm): direct DMA paths."""
    torch = pytest.importorskip("torch")
    raw = W.raw(500, 30000, 0.2, 0.5, n_wall=600)
    nodes = np.vstack([raw["vol"], raw["wall"]])
    surface = np.arange(len(raw["vol"]), len(nodes))
    d = gpu.build_distance_index(nodes, 3, surface)
    i0, v0 = oracle.update_volume(nodes, d, raw["ctrl"], raw["alpha"], 0.5, 0, "c2", 0.2)
    pin = lambda shape, dt: torch.empty(shape, dtype=dt, pin_memory=True).numpy()
    nodes_p, d_p = pin(nodes.shape, torch.float64), pin(d.shape, torch.float64)
    nodes_p[:], d_p[:] = nodes, d
    out = (pin((len(nodes),), torch.int64).view(np.uint64), pin((len(nodes), 3), torch.float64))
    chunked(6000)
    i1, v1 = gpu.update_volume(nodes_p, d_p, raw["ctrl"], raw["alpha"], 0.5, 0, "c2", 0.2,
                               capi.EXACT, out=out)
    assert np.array_equal(i0, i1) and np.array_equal(v0, v1)


def test_pipelined_nothing_active(gpu, chunked):
    rng = np.random.default_rng(5)
    nodes = rng.random((20000, 3)) + 10.0
    d = np.full(len(nodes), 5.0)
    chunked(3000)
    i, v = gpu.update_volume(nodes, d, rng.random((50, 3)), rng.random((50, 3)), 1.0, 0, "c2",
                             0.5, capi.EXACT)
    assert len(i) == 0 and len(v) == 0
