"""CholeskyFactor (rbf.hpp:41-60, rbf.cpp:71-121) and assemble_surface_matrix
(rbf.hpp:35-36, rbf.cpp:56-69) on the device, against the reference's own
class and function (oracle/_ref) and the known answers of
proj/tests/test_rbf.cpp:82-94 and :183-221."""
import os

import numpy as np
import pytest

from paper_2107_13887_b200 import capi

pytestmark = pytest.mark.gpu


def test_surface_matrix_kats(gpu):  # test_rbf.cpp:82-94
    assert np.array_equal(gpu.assemble_surface_matrix([(0, 0, 0), (1, 0, 0)], "c2", 2.0),
                          [[1.0, 0.1875], [0.1875, 1.0]])
    assert np.array_equal(gpu.assemble_surface_matrix([(3, 4, 0)], "c2", 2.0), [[1.0]])
    assert np.array_equal(gpu.assemble_surface_matrix([(0, 0, 0), (2.5, 0, 0)], "c2", 2.0),
                          [[1.0, 0.0], [0.0, 1.0]])


@pytest.mark.parametrize("kind", ["c0", "c2", "c4", "c6"])
def test_surface_matrix_matches_reference(gpu, ref, kind):
    rng = np.random.default_rng(5)
    p = rng.random((300, 3))
    assert np.array_equal(gpu.assemble_surface_matrix(p, kind, 0.7),
                          ref.assemble_surface_matrix(p, kind, 0.7))


def _columns(points, R, kind="c2"):
    """rbf.cpp:165-171: column k = phi(|p_j - p_k|) for j < k, then 1.0."""
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(__file__)), "oracle"))
    import pyoracle

    o = pyoracle.Oracle("port")
    for k in range(len(points)):
        d = np.sqrt(((points[:k] - points[k]) ** 2).sum(axis=1)) if k else np.zeros(0)
        col = np.array([o.eval_wendland(kind, x / R) for x in d] + [1.0])
        yield col


@pytest.mark.parametrize("n,dim", [(25, 2), (400, 3), (1500, 3)])
def test_incremental_factor_matches_reference(gpu, ref, n, dim):
    """test_rbf.cpp:183-213: rows appended one at a time, then one solve --
    bit-identical to the reference class (x, size, smallest_pivot), and within
    1e-10 of a dense solve."""
    rng = np.random.default_rng(31 + n)
    pts = rng.random((n, 3)) * 0.8
    if dim == 2:
        pts[:, 2] = 0.0
    f, g = gpu.cholesky(), ref.cholesky()
    for col in _columns(pts, 0.8):
        f.append(col)
        g.append(col)
    assert f.size() == g.size() == n
    assert f.smallest_pivot() == g.smallest_pivot()
    rhs = np.sin(1.7 * np.arange(n))
    x = f.solve(rhs)
    assert np.array_equal(x, g.solve(rhs))
    A = gpu.assemble_surface_matrix(pts, "c2", 0.8)
    assert np.abs(A @ x - rhs).max() <= 1e-8 * np.abs(rhs).max()


def test_factor_global_memory_variant(gpu, ref, monkeypatch):
    """The append / forward substitution for factors beyond shared memory
    (L and the row streamed from global memory), forced at a small size."""
    monkeypatch.setenv("IMB_INSERT_RING0", "1")
    rng = np.random.default_rng(8)
    pts = rng.random((300, 3))
    f, g = gpu.cholesky(), ref.cholesky()
    for col in _columns(pts, 0.9):
        f.append(col)
        g.append(col)
    rhs = rng.standard_normal(300)
    assert np.array_equal(f.solve(rhs), g.solve(rhs))


def test_factor_errors_and_state(gpu, ref):
    f, g = gpu.cholesky(), ref.cholesky()
    with pytest.raises(ValueError, match="column length must be current size \\+ 1"):
        f.append([1.0, 2.0])
    f.append([1.0]), g.append([1.0])
    with pytest.raises(ValueError, match="rhs size does not match factorization"):
        f.solve([1.0, 2.0])
    # a failed append leaves the factor unchanged but keeps the raised max
    # diagonal (rbf.cpp:89-96): pivot^2 = 4 - 2^2 = 0 fails with max_diag 4 ...
    with pytest.raises(capi.SolveError) as e:
        f.append([2.0, 4.0])
    with pytest.raises(Exception) as e2:
        g.append([2.0, 4.0])
    assert str(e.value) == str(e2.value)
    assert "matrix not numerically positive definite at row 1" in str(e.value)
    assert f.size() == g.size() == 1
    # ... so a pivot of 2e-14 now fails (1e-14 * 4), as in the reference
    col = [0.0, 4e-28]
    with pytest.raises(capi.SolveError):
        f.append(col)
    with pytest.raises(Exception):
        g.append(col)
    f.append([0.5, 1.0]), g.append([0.5, 1.0])
    assert f.size() == g.size() == 2 and f.smallest_pivot() == g.smallest_pivot()
    assert np.array_equal(f.solve([1.0, -1.0]), g.solve([1.0, -1.0]))


def test_two_point_kat(gpu):  # test_rbf.cpp:96-119 through the class
    f = gpu.cholesky()
    f.append([1.0])
    f.append([0.1875, 1.0])
    x = f.solve([1.0, 0.0])
    b = 0.1875
    assert abs(x[0] - 1.0 / (1.0 - b * b)) <= 1e-12 and abs(x[1] + b / (1.0 - b * b)) <= 1e-12
