"""The speculative pipelined greedy (greedy_spec.cu) against the sequential
engine (IMB_SPEC=0) and the reference: identical control indices, alpha,
convergence record and residual whatever the number of chains in flight
(IMB_SPEC_S: 1 forces every chain to wait for its slot, 3 keeps a shallow
pipeline, the default a deep one), on a mirror-symmetric airfoil whose
near-ties make the predictor miss (rollbacks) and on a 3-D cloud."""
import numpy as np
import pytest

from paper_2107_13887_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _same(a, b):
    assert len(a.levels) == len(b.levels)
    for x, y in zip(a.levels, b.levels):
        assert np.array_equal(x.control_indices, y.control_indices)
        assert np.array_equal(x.alpha, y.alpha)
        assert np.array_equal(x.record_error, y.record_error)
        assert x.cap_hit == y.cap_hit
    assert np.array_equal(a.final_residual, b.final_residual)


def _cases():
    w = W.cfg2(0.3)
    yield "airfoil", w.nodes[w.surface], w.displacement, w.tol, 2, 600, w.R
    rng = np.random.default_rng(41)
    p = rng.random((2500, 3))
    d = np.stack([np.sin(3 * p[:, 0]), np.cos(2 * p[:, 1]), p[:, 2] ** 2], axis=1) * 0.01
    yield "cloud", p, d, 1e-4, 2, 700, 0.6


_REF = {}


@pytest.mark.parametrize("slots", ["1", "3", None])
def test_spec_equals_sequential_and_reference(gpu, oracle, monkeypatch, slots):
    for name, pos, disp, tol, levels, cap, R in _cases():
        monkeypatch.setenv("IMB_SPEC", "0")
        seq = gpu.run_multilevel(pos, disp, tol, levels, cap, "c2", R)
        monkeypatch.setenv("IMB_SPEC", "1")
        if slots:
            monkeypatch.setenv("IMB_SPEC_S", slots)
        spec = gpu.run_multilevel(pos, disp, tol, levels, cap, "c2", R)
        _same(seq, spec)
        if name not in _REF:
            _REF[name] = oracle.run_multilevel(pos, disp, tol, levels, cap, "c2", R)
        ref = _REF[name]
        for x, y in zip(spec.levels, ref.levels):
            assert np.array_equal(x.control_indices, y.control_indices), name
            assert np.array_equal(x.alpha, y.alpha), name


def test_spec_single_cta_predictor(gpu, oracle, monkeypatch):
    """The fallback predictor (single-CTA insert + fast solve, used when the
    cluster kernel's shared memory does not fit) gives the same selection."""
    monkeypatch.setenv("IMB_SPEC_NOCLUSTER", "1")
    w = W.cfg2(0.3)
    pos = w.nodes[w.surface]
    a = gpu.run_multilevel(pos, w.displacement, w.tol, 2, 600, "c2", w.R)
    b = oracle.run_multilevel(pos, w.displacement, w.tol, 2, 600, "c2", w.R)
    for x, y in zip(a.levels, b.levels):
        assert np.array_equal(x.control_indices, y.control_indices)
        assert np.array_equal(x.alpha, y.alpha)
