"""Small cases of every device path, for compute-sanitizer (one tool per
run: memcheck / racecheck / synccheck).  The greedy runs twice: the
sequential engine (k_insert / k_backward_t / k_sweep, IMB_SPEC=0) and the
speculative pipeline's kernels one at a time (IMB_SPEC_S=1 keeps a single
chain in flight).  Exit code 0 when every result still equals the oracle."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import pyoracle  # noqa: E402

from paper_2107_13887_b200 import capi, workloads as W  # noqa: E402


def main():
    spec = len(sys.argv) > 1 and sys.argv[1] == "spec"
    os.environ["IMB_SPEC"] = "1" if spec else "0"
    orc = pyoracle.Oracle("ref" if pyoracle.available("ref") else "port")
    ctx = capi.Context(0)
    w = W.cfg1(0.1)
    pos = w.nodes[w.surface]
    a = ctx.run_multilevel(pos, w.displacement, w.tol, 2, 60, "c2", w.R)
    b = orc.run_multilevel(pos, w.displacement, w.tol, 2, 60, "c2", w.R)
    for x, y in zip(a.levels, b.levels):
        assert np.array_equal(x.control_indices, y.control_indices) and np.array_equal(x.alpha, y.alpha)
    print("greedy ok", [len(l.control_indices) for l in a.levels], flush=True)
    if spec:
        return
    rng = np.random.default_rng(3)
    p = rng.random((90, 3))
    d = rng.standard_normal((90, 3))
    assert np.array_equal(ctx.solve_weights(p, d, "c2", 0.7), orc.solve_weights(p, d, "c2", 0.7))
    f, g = ctx.cholesky(), orc.cholesky() if orc.flavour == "ref" else None
    A = ctx.assemble_surface_matrix(p[:40], "c2", 0.7)
    for k in range(40):
        f.append(A[k, :k + 1])
    x = f.solve(np.ones(40))
    assert np.abs(A @ x - 1).max() < 1e-8
    print("rbf ok", flush=True)
    dist = ctx.build_distance_index(w.nodes, 2, w.surface)
    assert np.array_equal(dist, orc.build_distance_index(w.nodes, 2, w.surface))
    lv = a.levels[-1]
    for prec in (capi.EXACT, capi.FP64, capi.FP32):
        i1, v1 = ctx.update_volume(w.nodes, dist, pos[lv.control_indices], lv.alpha, w.D,
                                   w.psi_kind, "c2", w.R, prec)
    i0, v0 = orc.update_volume(w.nodes, dist, pos[lv.control_indices], lv.alpha, w.D, w.psi_kind,
                               "c2", w.R)
    i1, v1 = ctx.update_volume(w.nodes, dist, pos[lv.control_indices], lv.alpha, w.D, w.psi_kind,
                               "c2", w.R, capi.EXACT)
    assert np.array_equal(i0, i1) and np.array_equal(v0, v1)
    plan = capi.VolumePlan(ctx, w.nodes, 2, w.surface, cutoff=w.D)
    plan.set_level(0, pos[lv.control_indices], lv.alpha, w.D, w.psi_kind, "c2", w.R, capi.EXACT)
    plan.run_steps(1, "c2", w.R, capi.EXACT, flush_l2=False)
    plan.bench_passes(w.D, w.D, reps=1)
    print("volume ok", flush=True)


if __name__ == "__main__":
    main()
