"""Quick GPU parity probe (development aid): product C-ABI vs the oracle."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
from pyoracle import Oracle  # noqa: E402

from paper_2107_13887_b200 import capi, workloads as W  # noqa: E402

orc = Oracle("ref")
ctx = capi.Context(0)
rng = np.random.default_rng(1)
ok = True


def check(name, cond, extra=""):
    global ok
    ok &= bool(cond)
    print(("PASS " if cond else "FAIL ") + name, extra, flush=True)


# eval_interpolant exact vs reference
ctrl = rng.random((300, 3))
alpha = rng.standard_normal((300, 3))
q = rng.random((5000, 3)) * 2 - 0.5
for R in (0.05, 0.3, 1.0, 1e6):
    a = ctx.eval_interpolant(ctrl, alpha, "c2", R, q, capi.EXACT)
    b = orc.eval_interpolant(ctrl, alpha, "c2", R, q)
    check(f"eval_interpolant exact R={R}", np.array_equal(a, b), np.abs(a - b).max())
    f = ctx.eval_interpolant(ctrl, alpha, "c2", R, q, capi.FP64)
    err = np.abs(f - b).max() / max(np.abs(b).max(), 1e-300)
    check(f"eval_interpolant fast R={R}", err < 1e-12, err)

# wall distance
nodes = rng.random((20000, 3)) * 4 - 2
surf = np.arange(500)
t = time.time()
d1 = ctx.build_distance_index(nodes, 3, surf)
d2 = orc.build_distance_index(nodes, 3, surf)
check("build_distance_index 3D", np.array_equal(d1, d2), time.time() - t)
w = W.cfg1(0.5)
d1 = ctx.build_distance_index(w.nodes, 2, w.surface)
d2 = orc.build_distance_index(w.nodes, 2, w.surface)
check("build_distance_index cfg1/2", np.array_equal(d1, d2))

# update_volume
for psi in (0, 1):
    i1, v1 = ctx.update_volume(w.nodes, d2, ctrl[:50] * 0.3, alpha[:50], 0.4, psi, "c2", 0.5,
                               capi.EXACT)
    i2, v2 = orc.update_volume(w.nodes, d2, ctrl[:50] * 0.3, alpha[:50], 0.4, psi, "c2", 0.5)
    check(f"update_volume exact psi={psi}", np.array_equal(i1, i2) and np.array_equal(v1, v2),
          (len(i1), len(i2)))
    i1, v1 = ctx.update_volume(w.nodes, d2, ctrl[:50] * 0.3, alpha[:50], 0.4, psi, "c2", 0.5,
                               capi.FP64)
    err = np.abs(v1 - v2).max() / np.abs(v2).max()
    check(f"update_volume fast psi={psi}", np.array_equal(i1, i2) and err < 1e-10, err)

# greedy
pos = w.nodes[w.surface]
t = time.time()
g1 = ctx.greedy_level(pos, w.displacement, 1e-3, 5000, "c2", 0.5)
t1 = time.time() - t
t = time.time()
g2 = orc.greedy_level(pos, w.displacement, 1e-3, 5000, "c2", 0.5)
t2 = time.time() - t
check("greedy_level indices", np.array_equal(g1.control_indices, g2.control_indices),
      (len(g1.control_indices), len(g2.control_indices), t1, t2))
check("greedy_level alpha", np.array_equal(g1.alpha, g2.alpha))
check("greedy_level residual", np.array_equal(g1.residual, g2.residual))
check("greedy_level record", np.array_equal(g1.record_error, g2.record_error))

# solve_weights
p = rng.random((200, 3))
dsp = rng.standard_normal((200, 3))
a1 = ctx.solve_weights(p, dsp, "c2", 0.4)
a2 = orc.solve_weights(p, dsp, "c2", 0.4)
check("solve_weights", np.array_equal(a1, a2))
try:
    ctx.solve_weights([[0, 0, 0], [1e-18, 0, 0]], [[1, 0, 0], [2, 0, 0]], "c2", 1.0)
    check("solve_weights SolveError", False)
except capi.SolveError as e:
    check("solve_weights SolveError", "points 0 and 1" in str(e), str(e))

# multilevel + deform cfg1
w = W.cfg1()
pos = w.nodes[w.surface]
t = time.time()
m1 = ctx.run_multilevel(pos, w.displacement, w.tol, w.levels, w.cap, w.kind, w.R)
t1 = time.time() - t
t = time.time()
m2 = orc.run_multilevel(pos, w.displacement, w.tol, w.levels, w.cap, w.kind, w.R)
t2 = time.time() - t
same = len(m1.levels) == len(m2.levels) and all(
    np.array_equal(a.control_indices, b.control_indices) and np.array_equal(a.alpha, b.alpha)
    for a, b in zip(m1.levels, m2.levels))
check("run_multilevel cfg1", same and np.array_equal(m1.final_residual, m2.final_residual),
      ([len(l.control_indices) for l in m1.levels], t1, t2))

t = time.time()
r1 = ctx.deform(w.nodes, 2, w.surface, w.displacement, (), w.tol, w.levels, w.cap, w.kind, w.R,
                5.0, -1.0, 0, capi.EXACT)
t1 = time.time() - t
t = time.time()
r2 = orc.deform(w.nodes, 2, w.surface, w.displacement, (), w.tol, w.levels, w.cap, w.kind, w.R,
                5.0)
t2 = time.time() - t
check("deform cfg1 exact", np.array_equal(r1["nodes"], r2["nodes"]) and
      np.array_equal(r1["touched"], r2["touched"]), (t1, t2, r1["touched"], r2["touched"]))
r3 = ctx.deform(w.nodes, 2, w.surface, w.displacement, (), w.tol, w.levels, w.cap, w.kind, w.R,
                5.0, -1.0, 0, capi.FP64)
dv1 = r3["nodes"] - w.nodes
dv2 = r2["nodes"] - w.nodes
err = np.abs(dv1 - dv2).max() / np.abs(dv2).max()
check("deform cfg1 fast", err < 1e-10, (err, r3["total_seconds"], r3["greedy_seconds"],
                                         r3["distance_seconds"], r3["volume_seconds"]))
print("ALL OK" if ok else "SOME FAILED")
